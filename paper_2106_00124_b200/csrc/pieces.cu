// pieces.cu -- the reference's building blocks as device kernels, for callers
// that compose them directly:
//
//   k_add_contribution  add_contribution(src, dst, dim, offset)  excluded.py:111-126
//                       dst[.., x_dim, ..] (+)= src_slice[x_dim + offset, ..] where
//                       in range, broadcast over the dims before dim (accumulates)
//   k_elementwise       MonoidOps.combine_into / rcombine_into / subtract_into /
//                       rsubtract_scalar (monoid.py:145-159, 184-198, 219-227,
//                       274-282), mod-add reducing after each operation
//
// Scans along an axis (MonoidOps.accumulate, prefix/suffix_along_dim) reuse the
// sequential scan kernels of sat.cu; fold reuses the deterministic total of
// reduce_excl.cu.  All of these are plain streaming element maps (2-3 N s).
#include <type_traits>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

namespace {

__device__ __forceinline__ i64 fmod_dev(i64 v, const FastMod& fm) {
  const unsigned long long u = v >= 0 ? (unsigned long long)v : (unsigned long long)(-(v + 1));
  const unsigned long long q = __umul64hi(u, fm.inv);
  unsigned long long r = u - q * fm.m;
  while (r >= fm.m) r -= fm.m;
  return v >= 0 ? (i64)r : (i64)(fm.m - 1 - r);
}

// one combine / subtract with the operator's semantics (MOD: np.add or
// np.subtract on int64, then np.remainder)
template <class T, class Op, bool MOD>
__device__ __forceinline__ T combine(T a, T b, const FastMod& fm) {
  if constexpr (MOD) return (T)fmod_dev(OpAdd::apply<i64>((i64)a, (i64)b), fm);
  return Op::apply(a, b);
}
template <class T, class Op, bool MOD>
__device__ __forceinline__ T subtract(T a, T b, const FastMod& fm) {
  if constexpr (MOD) return (T)fmod_dev(OpAdd::inverse<i64>((i64)a, (i64)b), fm);
  return OpAdd::inverse<T>(a, b);
}

}  // namespace

template <class T, class Op, bool MOD>
__global__ void k_add_contribution(const T* __restrict__ src, T* __restrict__ dst, int64_t outer,
                                   int64_t n, int64_t inner, int64_t offset, FastMod fm) {
  const int64_t lo = offset < 0 ? -offset : 0;
  const int64_t hi = n - offset < n ? n - offset : n;
  if (lo >= hi) return;
  const int64_t span = (hi - lo) * inner;
  const int64_t total = outer * span;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / span;
    const int64_t rem = e - o * span;  // (x - lo) * inner + m
    const int64_t x = lo + rem / inner;
    const int64_t m = rem - (x - lo) * inner;
    T* p = dst + (o * n + x) * inner + m;
    *p = combine<T, Op, MOD>(*p, src[(x + offset) * inner + m], fm);
  }
}

// kind 0: dst = dst (+) src;  kind 1: dst = dst (-) src;  kind 2: dst = s (-) dst
template <class T, class Op, bool MOD>
__global__ void k_elementwise(T* __restrict__ dst, const T* __restrict__ src, T scalar, int kind,
                              int64_t n, FastMod fm) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const T d = dst[e];
    T r;
    if (kind == 0) {
      r = combine<T, Op, MOD>(d, src[e], fm);
    } else if (kind == 1) {
      r = subtract<T, Op, MOD>(d, src[e], fm);
    } else {
      r = subtract<T, Op, MOD>(scalar, d, fm);
    }
    dst[e] = r;
  }
}

// The fold's result in the element type (float32 totals accumulate in float64;
// mod-add reduces the wrapping int64 sum, ModAddOps.fold).
template <class T, bool MOD>
__global__ void k_fold_result(const typename AccOf<T>::type* __restrict__ acc, T* __restrict__ out,
                              FastMod fm) {
  if constexpr (MOD) {
    *out = (T)fmod_dev((i64)*acc, fm);
  } else {
    *out = (T)*acc;
  }
}

namespace {

unsigned grid_of(int64_t work) {
  int64_t g = (work + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

#define EXSUM_DISPATCH_OPS(LAUNCH)                                        \
  if (op == 2) {                                                          \
    if (dtype != 2) return -1;                                            \
    LAUNCH(i64, OpAdd, true);                                             \
  }                                                                       \
  if (op == 1) {                                                          \
    if (dtype != 2) return -1;                                            \
    LAUNCH(i64, OpMax, false);                                            \
  }                                                                       \
  switch (dtype) {                                                        \
    case 0: LAUNCH(float, OpAdd, false);                                  \
    case 1: LAUNCH(double, OpAdd, false);                                 \
    case 2: LAUNCH(i64, OpAdd, false);                                    \
  }                                                                       \
  return -1;

int launch_add_contribution(int dtype, int op, const FastMod& fm, const void* src, void* dst,
                            int64_t outer, int64_t n, int64_t inner, int64_t offset,
                            cudaStream_t s) {
  const unsigned g = grid_of(outer * n * inner);
#define L(T, OP, MOD)                                                                        \
  k_add_contribution<T, OP, MOD><<<g, 256, 0, s>>>((const T*)src, (T*)dst, outer, n, inner,  \
                                                    offset, fm);                             \
  return 1;
  EXSUM_DISPATCH_OPS(L)
#undef L
}

int launch_elementwise(int dtype, int op, const FastMod& fm, void* dst, const void* src,
                       const void* scalar_host, int kind, int64_t n, cudaStream_t s) {
  const unsigned g = grid_of(n);
#define L(T, OP, MOD)                                                                      \
  {                                                                                        \
    T sc = T(0);                                                                           \
    if (scalar_host) sc = *(const T*)scalar_host;                                          \
    k_elementwise<T, OP, MOD><<<g, 256, 0, s>>>((T*)dst, (const T*)src, sc, kind, n, fm);  \
    return 1;                                                                              \
  }
  EXSUM_DISPATCH_OPS(L)
#undef L
}

int launch_fold_result(int dtype, int op, const FastMod& fm, const void* acc, void* out,
                       cudaStream_t s) {
  switch (dtype) {
    case 0: k_fold_result<float, false><<<1, 1, 0, s>>>((const double*)acc, (float*)out, fm); return 1;
    case 1: k_fold_result<double, false><<<1, 1, 0, s>>>((const double*)acc, (double*)out, fm); return 1;
    case 2:
      if (op == 2) {
        k_fold_result<i64, true><<<1, 1, 0, s>>>((const i64*)acc, (i64*)out, fm);
      } else {
        k_fold_result<i64, false><<<1, 1, 0, s>>>((const i64*)acc, (i64*)out, fm);
      }
      return 1;
  }
  return -1;
}

#undef EXSUM_DISPATCH_OPS

}  // namespace exsum
