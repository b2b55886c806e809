// reduce_excl.cu -- reductions and the box-complement row round.
//
//  * k_total / k_total_final: MonoidOps.fold (monoid.py:161-164, 200-204) for
//    BDBSC (excluded.py:72-75).  Two fixed-shape stages (per-CTA partials, then
//    one CTA in a fixed order), so the total is deterministic run to run.
//    float32 folds in float64: the reference's float32 sequential fold stalls
//    at 2^24, so parity for float32 is against the float64
//    upcast; the result is rounded to float32 once, like float(total) in
//    rsubtract_scalar (monoid.py:193-194).
//  * k_complement: out = total (-) in, for a BDBSC route with no windowed pass.
//  * k_row_reduce: R = (+)-reduction over the last axis (the dimension the
//    box-complement round peels, see box_complement in exsum_capi.cu).
//  * k_excl_rows: one box-complement round along the last axis:
//    out[r,x] = P[r,x-1] (+) S[r,x+k] (+) T[r], the "below"/"above" slabs of
//    add_contribution (excluded.py:111-126, 151-156) with P/S full-row
//    prefix/suffix of the windowed array W.  A warp owns a row: pass 1 runs
//    the suffix scan right to left (warp log-step scan + carry) into shared
//    memory, pass 2 runs the prefix left to right and combines.  The second
//    read of the row hits L2 (the row was read microseconds earlier), so HBM
//    sees one read and one write per element.
#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

constexpr int kTotalBlocks = 1184;  // 8 CTAs per SM on 148 SMs; fixed => deterministic
constexpr int kPartialsCap = 16384;  // capacity of the partials workspace (fused totals)

template <class Acc, class Op>
__device__ __forceinline__ Acc warp_reduce(Acc v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = Op::apply(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

// Every CTA folds one contiguous range whose length is a multiple of the
// 16-byte vector, with four vectors of loads in flight per thread (a scalar
// load per thread and iteration read 2.7 TB/s on a 64 MB float32 array and
// 5.8 TB/s on 1 GB of float64; this form 6.2+ TB/s).  The shape of the fold
// (range per CTA, strides, four accumulators folded in a fixed order) depends
// only on N and the grid, so the total stays deterministic run to run.
template <class T, class Op>
__global__ void __launch_bounds__(256)
k_total(const T* __restrict__ in, int64_t N, typename AccOf<T>::type* __restrict__ partials) {
  typedef typename AccOf<T>::type Acc;
  constexpr int VE = 16 / sizeof(T);
  __shared__ Acc sh[8];
  Acc a0 = Op::template identity<Acc>(), a1 = a0, a2 = a0, a3 = a0;
  int64_t per = (N + gridDim.x - 1) / gridDim.x;
  per = (per + VE - 1) / VE * VE;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < N ? lo + per : N;
  if (lo < hi) {
    if (((uintptr_t)in % 16) == 0) {
      const int64_t nv = (hi - lo) / VE;  // whole vectors of this range
      const T* p = in + lo;
      int64_t i = threadIdx.x;
      for (; i + 3 * 256 < nv; i += 4 * 256) {
        const Vec<T, VE> v0 = ld_stream<T, VE>(p + i * VE);
        const Vec<T, VE> v1 = ld_stream<T, VE>(p + (i + 256) * VE);
        const Vec<T, VE> v2 = ld_stream<T, VE>(p + (i + 512) * VE);
        const Vec<T, VE> v3 = ld_stream<T, VE>(p + (i + 768) * VE);
#pragma unroll
        for (int j = 0; j < VE; ++j) {
          a0 = Op::apply(a0, (Acc)v0.v[j]);
          a1 = Op::apply(a1, (Acc)v1.v[j]);
          a2 = Op::apply(a2, (Acc)v2.v[j]);
          a3 = Op::apply(a3, (Acc)v3.v[j]);
        }
      }
      for (; i < nv; i += 256) {
        const Vec<T, VE> v0 = ld_stream<T, VE>(p + i * VE);
#pragma unroll
        for (int j = 0; j < VE; ++j) a0 = Op::apply(a0, (Acc)v0.v[j]);
      }
      for (int64_t x = lo + nv * VE + threadIdx.x; x < hi; x += 256)  // the array's last elements
        a1 = Op::apply(a1, (Acc)ld1(in + x));
    } else {
      for (int64_t x = lo + threadIdx.x; x < hi; x += 256) a0 = Op::apply(a0, (Acc)ld1(in + x));
    }
  }
  Acc acc = Op::apply(Op::apply(a0, a1), Op::apply(a2, a3));
  acc = warp_reduce<Acc, Op>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = Op::apply(t, sh[w]);
    partials[blockIdx.x] = t;
  }
}

template <class Acc, class Op>
__global__ void k_total_final(const Acc* __restrict__ partials, int np, Acc* __restrict__ total) {
  __shared__ Acc sh[32];
  Acc acc = Op::template identity<Acc>();
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc = Op::apply(acc, partials[i]);
  acc = warp_reduce<Acc, Op>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = sh[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = Op::apply(t, sh[w]);
    *total = t;
  }
}

template <class T>
__global__ void k_complement(const T* __restrict__ in, T* __restrict__ out, int64_t N,
                             const typename AccOf<T>::type* __restrict__ total) {
  const T tot = (T)(*total);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    st1(out + i, OpAdd::inverse<T>(tot, ld1(in + i)));
}

// R[r] = fold of row r; warp per row (n >= 32) or thread per row (short rows)
template <class T, class Op>
__global__ void __launch_bounds__(256)
k_row_reduce(const T* __restrict__ in, T* __restrict__ R, int64_t rows, int64_t n) {
  typedef typename AccOf<T>::type Acc;
  if (n >= 32) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < rows; r += nwarps) {
      const T* p = in + r * n;
      Acc acc = Op::template identity<Acc>();
      for (int64_t x = lane; x < n; x += 32) acc = Op::apply(acc, (Acc)ld1(p + x));
      acc = warp_reduce<Acc, Op>(acc);
      if (lane == 0) R[r] = (T)acc;
    }
  } else {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
      const T* p = in + r * n;
      Acc acc = (Acc)p[0];
      for (int64_t x = 1; x < n; ++x) acc = Op::apply(acc, (Acc)p[x]);
      R[r] = (T)acc;
    }
  }
}

// inclusive warp scans (log-step), identity-padded outside [0, valid)
template <class T, class Op>
__device__ __forceinline__ T warp_incl_prefix(T v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v = Op::apply(t, v);
  }
  return v;
}
template <class T, class Op>
__device__ __forceinline__ T warp_incl_suffix(T v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T t = __shfl_down_sync(0xffffffffu, v, d);
    if (lane + d < 32) v = Op::apply(v, t);
  }
  return v;
}

// S buffer per warp: shared memory when the row fits (SMEM), else global.
template <class T, class Op, bool SMEM>
__global__ void __launch_bounds__(128)
k_excl_rows(const T* __restrict__ W, T* __restrict__ out, const T* __restrict__ Tail,
            int64_t rows, int64_t n, int64_t k, T* __restrict__ gS) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T ident = Op::template identity<T>();
  const int64_t nsteps = (n + 31) / 32;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const T* pw = W + r * n;
    T* po = out + r * n;
    T* S = SMEM ? reinterpret_cast<T*>(smem_raw) + (int64_t)wib * n : gS + r * n;
    // pass 1: full-row inclusive suffix, right to left
    T carry = ident;
    for (int64_t s = nsteps - 1; s >= 0; --s) {
      const int64_t x = s * 32 + lane;
      T v = x < n ? pw[x] : ident;
      v = warp_incl_suffix<T, Op>(v, lane);
      v = Op::apply(v, carry);
      carry = __shfl_sync(0xffffffffu, v, 0);
      if (x < n) S[x] = v;
    }
    __syncwarp();
    const T tail = Tail ? Tail[r] : ident;
    const bool has_tail = Tail != nullptr;
    // pass 2: exclusive prefix left to right, combine the two slabs
    T pcarry = ident;  // P[x0 - 1]
    for (int64_t s = 0; s < nsteps; ++s) {
      const int64_t x = s * 32 + lane;
      T v = x < n ? ld1(pw + x) : ident;
      const T incl = Op::apply(pcarry, warp_incl_prefix<T, Op>(v, lane));
      T excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = pcarry;
      pcarry = __shfl_sync(0xffffffffu, incl, 31);
      if (x < n) {
        T o = ident;
        bool any = false;
        if (x >= 1) { o = excl; any = true; }
        if (x + k < n) { o = any ? Op::apply(o, S[x + k]) : S[x + k]; any = true; }
        if (has_tail) o = any ? Op::apply(o, tail) : tail;
        st1(po + x, o);
      }
    }
    __syncwarp();
  }
}

// Rows of n <= 32*C elements: a warp owns a row, lane l owns elements
// [lC, lC+C) in registers.  The row is staged through shared memory with
// coalesced 16-byte loads (chunk stride C+VE keeps vector alignment and
// spreads the lanes over all banks), then: lane-local fold -> warp-level
// exclusive prefix/suffix of the lane totals -> per-element S into a second,
// scalar-padded buffer (read back at the shifted position x+k) -> P carried in
// a register.  Out-of-range terms are the identity (x (+) e == x, so this is
// the reference's "leave untouched").  One read and one write of W per
// element, ~0.4 warp instructions per element.
template <class T, class Op, int C, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
k_excl_rows_reg(const T* __restrict__ W, T* __restrict__ out, const T* __restrict__ Tail,
                int64_t rows, int64_t n, int64_t k) {
  constexpr int VE = 16 / sizeof(T);
  constexpr int CV = C >= VE ? C / VE : 1;
  constexpr int SA = C >= VE ? C + VE : C + 1;  // raw/out chunk stride
  constexpr int SB = C + 1;                      // S chunk stride (odd)
  typedef Vec<T, VE> VT;
  __shared__ __align__(16) T smem[WARPS][32 * SA + 32 * SB];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  T* sa = smem[wib];
  T* sb = smem[wib] + 32 * SA;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T ident = Op::template identity<T>();
  const bool vec = C >= VE && n == 32 * C && ((uintptr_t)W % 16) == 0 && ((uintptr_t)out % 16) == 0;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const T* pw = W + r * n;
    T* po = out + r * n;
    if (vec) {
#pragma unroll
      for (int i = 0; i < CV; ++i) {
        const int v = i * 32 + lane;
        *reinterpret_cast<VT*>(sa + (v / CV) * SA + (v % CV) * VE) = ld_stream<T, VE>(pw + v * VE);
      }
    } else {
      for (int v = lane; v < 32 * C; v += 32) sa[(v / C) * SA + v % C] = v < n ? ld1(pw + v) : ident;
    }
    __syncwarp();
    T a[C];
#pragma unroll
    for (int j = 0; j < C; ++j) a[j] = sa[lane * SA + j];
    T tot = a[0];
#pragma unroll
    for (int j = 1; j < C; ++j) tot = Op::apply(tot, a[j]);
    T pin = tot, sin = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T tp = __shfl_up_sync(0xffffffffu, pin, d);
      const T ts = __shfl_down_sync(0xffffffffu, sin, d);
      if (lane >= d) pin = Op::apply(tp, pin);
      if (lane + d < 32) sin = Op::apply(sin, ts);
    }
    T pre = __shfl_up_sync(0xffffffffu, pin, 1);
    T suf = __shfl_down_sync(0xffffffffu, sin, 1);
    if (lane == 0) pre = ident;
    if (lane == 31) suf = ident;
    T run = suf;
#pragma unroll
    for (int j = C - 1; j >= 0; --j) {
      run = Op::apply(a[j], run);
      sb[lane * SB + j] = run;
    }
    __syncwarp();
    const T tail = Tail ? Tail[r] : ident;
    T pe = pre;  // P[x-1]; the identity at x == 0
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int64_t y = (int64_t)lane * C + j + k;
      const T sv = y < n ? sb[(y / C) * SB + (y % C)] : ident;
      const T o = Op::apply(Op::apply(pe, sv), tail);
      pe = Op::apply(pe, a[j]);
      a[j] = o;
    }
#pragma unroll
    for (int j = 0; j < C; ++j) sa[lane * SA + j] = a[j];
    __syncwarp();
    if (vec) {
#pragma unroll
      for (int i = 0; i < CV; ++i) {
        const int v = i * 32 + lane;
        st_stream<T, VE>(po + v * VE, *reinterpret_cast<const VT*>(sa + (v / CV) * SA + (v % CV) * VE));
      }
    } else {
      for (int v = lane; v < n; v += 32) st1(po + v, sa[(v / C) * SA + v % C]);
    }
    __syncwarp();
  }
}

namespace {

template <class T, class Op>
int go_total(const T* in, int64_t N, void* partials, void* total, cudaStream_t s) {
  typedef typename AccOf<T>::type Acc;
  k_total<T, Op><<<kTotalBlocks, 256, 0, s>>>(in, N, (Acc*)partials);
  k_total_final<Acc, Op><<<1, 1024, 0, s>>>((const Acc*)partials, kTotalBlocks, (Acc*)total);
  return 2;
}

template <class T, class Op>
int go_row_reduce(const T* in, T* R, int64_t rows, int64_t n, cudaStream_t s) {
  int64_t threads = n >= 32 ? rows * 32 : rows;
  int64_t grid = (threads + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  k_row_reduce<T, Op><<<(unsigned)grid, 256, 0, s>>>(in, R, rows, n);
  return 1;
}

constexpr size_t kExclSmemPerWarpMax = 48 * 1024;

template <class T, class Op, int C>
int go_excl_reg(const T* W, T* out, const T* Tail, int64_t rows, int64_t n, int64_t k,
                cudaStream_t s) {
  constexpr int VE = 16 / sizeof(T);
  constexpr int SA = C >= VE ? C + VE : C + 1;
  constexpr size_t PER_WARP = (size_t)32 * (SA + C + 1) * sizeof(T);
  constexpr int WARPS = PER_WARP * 4 <= 48 * 1024 ? 4 : (PER_WARP * 2 <= 48 * 1024 ? 2 : 1);
  int64_t grid = (rows + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  k_excl_rows_reg<T, Op, C, WARPS><<<(unsigned)grid, WARPS * 32, 0, s>>>(W, out, Tail, rows, n, k);
  return 1;
}

template <class T, class Op>
int go_excl(const T* W, T* out, const T* Tail, int64_t rows, int64_t n, int64_t k, T* scratch,
            cudaStream_t s) {
  if (n <= 32) return go_excl_reg<T, Op, 1>(W, out, Tail, rows, n, k, s);
  if (n <= 64) return go_excl_reg<T, Op, 2>(W, out, Tail, rows, n, k, s);
  if (n <= 128) return go_excl_reg<T, Op, 4>(W, out, Tail, rows, n, k, s);
  if (n <= 256) return go_excl_reg<T, Op, 8>(W, out, Tail, rows, n, k, s);
  if (n <= 512) return go_excl_reg<T, Op, 16>(W, out, Tail, rows, n, k, s);
  if (n <= 1024) return go_excl_reg<T, Op, 32>(W, out, Tail, rows, n, k, s);
  const size_t row_bytes = (size_t)n * sizeof(T);
  int64_t grid = (rows * 32 + 127) / 128;
  if (row_bytes <= kExclSmemPerWarpMax) {
    const size_t smem = row_bytes * 4;
    if (smem > 48 * 1024)
      ensure_smem((const void*)k_excl_rows<T, Op, true>, smem);
    const int64_t cap = (int64_t)num_sms() * 16;
    if (grid > cap) grid = cap;
    k_excl_rows<T, Op, true><<<(unsigned)grid, 128, smem, s>>>(W, out, Tail, rows, n, k, nullptr);
  } else {
    const int64_t cap = (int64_t)num_sms() * 16;
    if (grid > cap) grid = cap;
    k_excl_rows<T, Op, false><<<(unsigned)grid, 128, 0, s>>>(W, out, Tail, rows, n, k, scratch);
  }
  return 1;
}

}  // namespace

int reduce_partials_count() { return kPartialsCap; }

// part is [rows][ppr] (written by k_axis_stream<EX=1> / k_strided_reg<..., EXTRA=1>)
template <class T, class Op>
__global__ void k_rowpart_final(const T* __restrict__ part, T* __restrict__ R, int64_t rows,
                                int64_t ppr) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    T acc = part[r * ppr];
    for (int64_t i = 1; i < ppr; ++i) acc = Op::apply(acc, part[r * ppr + i]);
    R[r] = acc;
  }
}

int launch_rowpart_final(int dtype, int op, const void* part, void* R, int64_t rows, int64_t ppr,
                         cudaStream_t s) {
  int64_t grid = (rows + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (dtype == F32 && op == ADD)
    k_rowpart_final<float, OpAdd><<<(unsigned)grid, 256, 0, s>>>((const float*)part, (float*)R, rows, ppr);
  else if (dtype == F64 && op == ADD)
    k_rowpart_final<double, OpAdd><<<(unsigned)grid, 256, 0, s>>>((const double*)part, (double*)R, rows, ppr);
  else if (dtype == I64 && op == ADD)
    k_rowpart_final<i64, OpAdd><<<(unsigned)grid, 256, 0, s>>>((const i64*)part, (i64*)R, rows, ppr);
  else if (dtype == I64 && op == MAX)
    k_rowpart_final<i64, OpMax><<<(unsigned)grid, 256, 0, s>>>((const i64*)part, (i64*)R, rows, ppr);
  else
    return -2;
  return 1;
}

int launch_total_final(int dtype, int op, const void* partials, int64_t np, void* total,
                       cudaStream_t s) {
  if (dtype == F32 || dtype == F64) {
    k_total_final<double, OpAdd><<<1, 1024, 0, s>>>((const double*)partials, (int)np, (double*)total);
  } else if (op == ADD) {
    k_total_final<i64, OpAdd><<<1, 1024, 0, s>>>((const i64*)partials, (int)np, (i64*)total);
  } else {
    k_total_final<i64, OpMax><<<1, 1024, 0, s>>>((const i64*)partials, (int)np, (i64*)total);
  }
  return 1;
}

int launch_total(int dtype, int op, const void* in, int64_t N, void* partials, void* total,
                 cudaStream_t s) {
  if (dtype == F32 && op == ADD) return go_total<float, OpAdd>((const float*)in, N, partials, total, s);
  if (dtype == F64 && op == ADD) return go_total<double, OpAdd>((const double*)in, N, partials, total, s);
  if (dtype == I64 && op == ADD) return go_total<i64, OpAdd>((const i64*)in, N, partials, total, s);
  if (dtype == I64 && op == MAX) return go_total<i64, OpMax>((const i64*)in, N, partials, total, s);
  return -2;
}

int launch_complement(int dtype, const void* in, void* out, int64_t N, const void* total,
                      cudaStream_t s) {
  int64_t grid = (N + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (grid > cap) grid = cap;
  if (dtype == F32)
    k_complement<float><<<(unsigned)grid, 256, 0, s>>>((const float*)in, (float*)out, N, (const double*)total);
  else if (dtype == F64)
    k_complement<double><<<(unsigned)grid, 256, 0, s>>>((const double*)in, (double*)out, N, (const double*)total);
  else
    k_complement<i64><<<(unsigned)grid, 256, 0, s>>>((const i64*)in, (i64*)out, N, (const i64*)total);
  return 1;
}

int launch_row_reduce(int dtype, int op, const void* in, void* R, int64_t rows, int64_t n,
                      cudaStream_t s) {
  if (dtype == F32 && op == ADD) return go_row_reduce<float, OpAdd>((const float*)in, (float*)R, rows, n, s);
  if (dtype == F64 && op == ADD) return go_row_reduce<double, OpAdd>((const double*)in, (double*)R, rows, n, s);
  if (dtype == I64 && op == ADD) return go_row_reduce<i64, OpAdd>((const i64*)in, (i64*)R, rows, n, s);
  if (dtype == I64 && op == MAX) return go_row_reduce<i64, OpMax>((const i64*)in, (i64*)R, rows, n, s);
  return -2;
}

size_t excl_rows_scratch_elems(int dtype, int64_t rows, int64_t n) {
  return (size_t)n * dtype_size(dtype) <= kExclSmemPerWarpMax ? 0 : (size_t)(rows * n);
}

int launch_excl_rows(int dtype, int op, const void* W, void* out, const void* T, int64_t rows,
                     int64_t n, int64_t k, void* scratch, cudaStream_t s) {
  if (dtype == F32 && op == ADD)
    return go_excl<float, OpAdd>((const float*)W, (float*)out, (const float*)T, rows, n, k, (float*)scratch, s);
  if (dtype == F64 && op == ADD)
    return go_excl<double, OpAdd>((const double*)W, (double*)out, (const double*)T, rows, n, k, (double*)scratch, s);
  if (dtype == I64 && op == ADD)
    return go_excl<i64, OpAdd>((const i64*)W, (i64*)out, (const i64*)T, rows, n, k, (i64*)scratch, s);
  if (dtype == I64 && op == MAX)
    return go_excl<i64, OpMax>((const i64*)W, (i64*)out, (const i64*)T, rows, n, k, (i64*)scratch, s);
  return -2;
}

}  // namespace exsum
