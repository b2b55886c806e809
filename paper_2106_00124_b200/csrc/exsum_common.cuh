// exsum_common.cuh -- shared device-side vocabulary for the box-sum kernels.
//
// Operators mirror the reference monoids (pkg/src/exsum/monoid.py):
//   add-i64  IntAddOps    monoid.py:130-164  (wraps mod 2^64 like numpy)
//   add-f64  FloatAddOps  monoid.py:167-204
//   add-f32  (test-side float32 FloatAddOps)
//   max-i64  IntMaxOps    monoid.py:207-232  (identity INT64_MIN, no inverse)
// Every combine is IEEE round-to-nearest; nothing here is compiled with
// fast-math, and there are no multiplies for FMA contraction to touch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <tuple>
#include <vector>

namespace exsum {

typedef long long i64;

struct OpAdd {
  template <class T>
  __device__ __forceinline__ static T apply(T a, T b) { return a + b; }
  template <class T>
  __device__ __forceinline__ static T identity() { return T(0); }
  template <class T>
  __device__ __forceinline__ static T inverse(T total, T v) { return total - v; }
};

template <>
__device__ __forceinline__ i64 OpAdd::apply<i64>(i64 a, i64 b) {
  return (i64)((unsigned long long)a + (unsigned long long)b);
}
template <>
__device__ __forceinline__ i64 OpAdd::inverse<i64>(i64 total, i64 v) {
  return (i64)((unsigned long long)total - (unsigned long long)v);
}

struct OpMax {
  template <class T>
  __device__ __forceinline__ static T apply(T a, T b) { return a >= b ? a : b; }
  template <class T>
  __device__ __forceinline__ static T identity();
  template <class T>
  __device__ __forceinline__ static T inverse(T, T v) { return v; }  // never used (no inverse)
};
template <>
__device__ __forceinline__ i64 OpMax::identity<i64>() { return (i64)0x8000000000000000ULL; }

// Accumulator type for totals: float32 data folds in float64 (the reference's
// float32 sequential fold stalls at 2^24 -- SURVEY 8(c)); others fold in place.
template <class T> struct AccOf { typedef T type; };
template <> struct AccOf<float> { typedef double type; };

// ---------------------------------------------------------------- vectors --
template <class T, int V>
struct alignas(sizeof(T) * V) Vec {
  T v[V];
};

// Streaming (evict-first) global loads/stores: every element of a pass is
// read once and written once.
template <class T, int V>
__device__ __forceinline__ Vec<T, V> ld_stream(const T* p) {
  Vec<T, V> r;
  if constexpr (sizeof(T) * V == 16) {
    int4 q = __ldcs(reinterpret_cast<const int4*>(p));
    r = *reinterpret_cast<Vec<T, V>*>(&q);
  } else if constexpr (sizeof(T) * V == 8) {
    int2 q = __ldcs(reinterpret_cast<const int2*>(p));
    r = *reinterpret_cast<Vec<T, V>*>(&q);
  } else {
    static_assert(sizeof(T) * V == 4, "vector width");
    int q = __ldcs(reinterpret_cast<const int*>(p));
    r = *reinterpret_cast<Vec<T, V>*>(&q);
  }
  return r;
}

// EXSUM_ST_KEEP (measurement build): plain stores, so a small array's
// intermediate stays in L2 for the next launch of the route
#ifndef EXSUM_ST_KEEP
#define EXSUM_ST_KEEP 0
#endif
template <class T, int V>
__device__ __forceinline__ void st_stream(T* p, const Vec<T, V>& v) {
  if constexpr (EXSUM_ST_KEEP) {
    *reinterpret_cast<Vec<T, V>*>(p) = v;
  } else if constexpr (sizeof(T) * V == 16) {
    __stcs(reinterpret_cast<int4*>(p), *reinterpret_cast<const int4*>(&v));
  } else if constexpr (sizeof(T) * V == 8) {
    __stcs(reinterpret_cast<int2*>(p), *reinterpret_cast<const int2*>(&v));
  } else {
    static_assert(sizeof(T) * V == 4, "vector width");
    __stcs(reinterpret_cast<int*>(p), *reinterpret_cast<const int*>(&v));
  }
}

template <class T>
__device__ __forceinline__ T ld1(const T* p) { return __ldcs(p); }
template <>
__device__ __forceinline__ i64 ld1<i64>(const i64* p) {
  return (i64)__ldcs(reinterpret_cast<const long long*>(p));
}
template <class T>
__device__ __forceinline__ void st1(T* p, T v) {
  if constexpr (EXSUM_ST_KEEP) *p = v;
  else __stcs(p, v);
}

// 64-bit-safe warp shuffles.
template <class T>
__device__ __forceinline__ T shfl_idx(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <class T>
__device__ __forceinline__ T shfl_down1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }
template <class T>
__device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }

// Epilogue applied at the final store of a route.  kind 0: plain store;
// kind 1: BDBSC complement out = total (-) v (excluded.py:72-75), with total
// read from device memory (double for float32, as AccOf).
template <class T>
struct Epilogue {
  const typename AccOf<T>::type* total;  // nullptr: plain store
  __device__ __forceinline__ T apply(T v) const {
    if (total == nullptr) return v;
    return OpAdd::inverse<T>((T)(*total), v);
  }
};

// Raise a kernel's dynamic shared-memory limit once per (kernel, device, size)
// instead of on every launch (cudaFuncSetAttribute costs microseconds of host
// time, which shows on small arrays).
inline void ensure_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::tuple<const void*, int, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  for (const auto& t : done)
    if (std::get<0>(t) == fn && std::get<1>(t) == dev && std::get<2>(t) >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  done.emplace_back(fn, dev, bytes);
}

// ------------------------------------------- bulk async copies (TMA path) --
// 1-D cp.async.bulk global->shared with mbarrier completion (sm_90+; SASS
// UBLKCP).  Sizes and addresses are multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Ampere-style per-thread async copies (LDGSTS), 16 bytes, L2 only.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_n(void* dst, const void* src) {
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace exsum
