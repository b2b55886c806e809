// tail2d.cu -- the box-complement tail of a 3-D array in two launches.
//
// The last-axis-first box-complement (exsum_capi.cu, route_box_complement)
// reduces A over its last axis into R (n0 x n1) and needs the tail
// T = BC(R, (k0, k1)) before its row round.  Restated for a 2-D R (the same
// recursion one level down, excluded.py:129-159 / SURVEY App. A.3):
//   R2[x0]     = (+)_{x1} R[x0, x1]                      (fold over R's last axis)
//   T1[x0]     = P2[x0 - 1] (+) S2[x0 + k0]              (1-D box complement of R2)
//   W[x0, x1]  = (+)_{y in [x0, min(x0+k0, n0))} R[y, x1]  (window along axis 0)
//   T[x0, x1]  = P_W[x0, x1 - 1] (+) S_W[x0, x1 + k1] (+) T1[x0]
// with P/S inclusive prefix/suffix and out-of-range terms the identity (an
// empty complement leaves the identity).  Every term is a fold of a subset of
// x's complement -- no inverse anywhere, so max is exact and float sums meet
// the strong route's bound.
//
// Before: rowpart_final + row_reduce + excl_rows (1 row) + fused_pair on R =
// four launches, each under-filled (C2: 21 us of a 130 us step).  Here:
//   k_tail_rows  one CTA per x0: R[x0, :] from the axis-0 pass's row partials
//                (or from R itself), written back, and R2[x0] by a block fold;
//   k_tail_block one CTA per k0-block of x0: T1 for its rows from R2 (two
//                block folds + <= 2 k0 sequential terms), the block's W rows
//                in shared memory from 2 k0 rows of R (in-block suffix, next
//                block's prefix -- each R element is read twice at most),
//                then a warp per row: suffix scan into a per-warp buffer, prefix
//                scan combined with S[x1 + k1] and T1, one store of T.
// Eligibility (tail2d_ok): the block tile k0 x n1 and the per-warp suffix
// buffers fit in shared memory.
#include <stdlib.h>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

namespace {

constexpr int kTailThreads = 256;
constexpr int kTailWarps = kTailThreads / 32;

template <class T, class Op>
__device__ __forceinline__ T block_fold(T v, T* sh) {
  // sh: kTailWarps elements; every thread gets the result
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = Op::apply(v, __shfl_xor_sync(0xffffffffu, v, d));
  __syncthreads();  // sh may still be read by a previous fold
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  T t = sh[0];
#pragma unroll
  for (int w = 1; w < kTailWarps; ++w) t = Op::apply(t, sh[w]);
  return t;
}

// part: [n0 * n1][ppr] row partials (ppr > 0) or nullptr (R already holds R).
// A CTA per x0 row of R, a thread per element of it: its ppr partials are
// contiguous, read as 16-byte vectors (consecutive threads on consecutive
// rows: the warp's loads cover one contiguous span), folded in order.
template <class T, class Op>
__global__ void __launch_bounds__(kTailThreads)
k_tail_rows(const T* __restrict__ part, int64_t ppr, T* __restrict__ R, T* __restrict__ R2,
            int64_t n0, int64_t n1) {
  __shared__ T sh[kTailWarps];
  constexpr int VE = 16 / sizeof(T);
  constexpr int PMAX = 16;  // partials per batch of loads
  for (int64_t x0 = blockIdx.x; x0 < n0; x0 += gridDim.x) {
    T acc = Op::template identity<T>();
    for (int64_t c = threadIdx.x; c < n1; c += blockDim.x) {
      const int64_t r = x0 * n1 + c;
      T v;
      if (part) {
        const T* pp = part + r * ppr;
        const bool vec = ppr % VE == 0;  // then every row's span is 16-byte aligned
        for (int64_t i0 = 0; i0 < ppr; i0 += PMAX) {
          T q[PMAX];
          const int cnt = (int)(ppr - i0 < PMAX ? ppr - i0 : PMAX);
          if (vec) {
#pragma unroll
            for (int w = 0; w < PMAX / VE; ++w)
              if (w * VE < cnt) {
                const Vec<T, VE> t = *reinterpret_cast<const Vec<T, VE>*>(pp + i0 + w * VE);
#pragma unroll
                for (int e = 0; e < VE; ++e) q[w * VE + e] = t.v[e];
              }
          } else {
#pragma unroll
            for (int i = 0; i < PMAX; ++i)
              if (i < cnt) q[i] = pp[i0 + i];
          }
          T t = i0 == 0 ? q[0] : Op::apply(v, q[0]);
#pragma unroll
          for (int i = 1; i < PMAX; ++i)
            if (i < cnt) t = Op::apply(t, q[i]);
          v = t;
        }
        R[r] = v;
      } else {
        v = R[r];
      }
      acc = Op::apply(acc, v);
    }
    acc = block_fold<T, Op>(acc, sh);
    if (threadIdx.x == 0) R2[x0] = acc;
  }
}

// One CTA per group of G = kGroup consecutive rows x0 of R (one warp per row):
//  * W rows: for the group [g0, g0+G) every window [x0, min(x0+k0, n0))
//    contains the common middle M = R[g0+G-1, min(g0+k0, n0)); then
//    W[g0+j] = A_j (+) M (+) B_j with A_j the rows [g0+j, g0+G-1) (an
//    in-group suffix) and B_j the rows [min(g0+k0,n0), min(g0+j+k0,n0)) (a
//    prefix past the middle): k0 + G - 1 row reads for G rows, thread per
//    column vector, every load of a column issued before its folds;
//  * T1 for the group from R2: two coalesced block folds of the common
//    prefix [0, g0) and suffix [min(g0+G-1+k0, n0), n0) plus <= G-1 terms
//    per row;
//  * row round: warp per row, lane per chunk of C (n1 <= 32 C) in
//    registers: chunk fold, warp scans of the chunk totals, the inclusive
//    suffix written to a padded shared row, the prefix walk combined with
//    S[x + k1] and T1 (out-of-range terms the identity), staged back and
//    stored coalesced.
constexpr int kGroup = 4;
constexpr int kGroupThreads = 256;  // the W phase and the folds; warps < kGroup run the row round
constexpr int kGroupWarps = kGroupThreads / 32;

template <int C>
__device__ __forceinline__ int poff(int x) { return (x / C) * (C + 1) + (x % C); }
template <int C>
__host__ __device__ constexpr int pitch() { return 32 * (C + 1); }

template <class T, class Op>
__device__ __forceinline__ T group_fold(T v, T* sh) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = Op::apply(v, __shfl_xor_sync(0xffffffffu, v, d));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  T t = sh[0];
#pragma unroll
  for (int w = 1; w < kGroupWarps; ++w) t = Op::apply(t, sh[w]);
  return t;
}

template <class T, class Op, int C>
__global__ void __launch_bounds__(kGroupThreads)
k_tail_group(const T* __restrict__ R, const T* __restrict__ R2, T* __restrict__ Tout, int n0,
             int n1, int k0, int k1, int gb, int ge) {
  // rows [gb, ge) of T (a shard: its own rows; R and Tout are indexed by the
  // global row, only rows >= gb are touched)
  constexpr int P = pitch<C>();
  constexpr int G = kGroup;
  __shared__ __align__(16) T Wt[G][P];
  __shared__ __align__(16) T Sr[G][P];
  __shared__ T t1[G];
  __shared__ T sh[kGroupWarps];
  const T ident = Op::template identity<T>();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int ngroups = (ge - gb + G - 1) / G;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int g0 = gb + grp * G;
    const int gm = ge - g0 < G ? ge - g0 : G;          // rows in this group
    const int gk = G <= k0 ? G : 1;                     // middle form needs G <= k0
    // ---- T1: P2[x0-1] (+) S2[x0+k0] for the group's rows ----
    T pre = ident;
    for (int y = threadIdx.x; y < g0; y += blockDim.x) pre = Op::apply(pre, R2[y]);
    pre = group_fold<T, Op>(pre, sh);
    const int s0 = g0 + gm - 1 + k0 < n0 ? g0 + gm - 1 + k0 : n0;
    T suf = ident;
    for (int y = s0 + threadIdx.x; y < n0; y += blockDim.x) suf = Op::apply(suf, R2[y]);
    suf = group_fold<T, Op>(suf, sh);
    if (threadIdx.x < gm) {
      const int x0 = g0 + threadIdx.x;
      T p = pre;
      for (int y = g0; y < x0; ++y) p = Op::apply(p, R2[y]);
      T q = suf;
      for (int y = x0 + k0; y < s0; ++y) q = Op::apply(q, R2[y]);
      t1[threadIdx.x] = Op::apply(p, q);
    }
    // ---- W rows of the group ----
    if (gk == G && gm == G) {
      const int mid_e = g0 + k0 < n0 ? g0 + k0 : n0;   // middle [g0+G-1, mid_e)
      const int mid_s = g0 + G - 1;
      // CW columns per thread at a time, every load of them issued before the
      // folds (the middle in batches of MB rows)
      constexpr int CW = 2;
      constexpr int MB = 16;
      for (int cb = threadIdx.x; cb < n1; cb += CW * blockDim.x) {
        T a[CW][G - 1], bq[CW][G - 1], mv[CW];
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          const int c = cb + u * blockDim.x;
          const bool ok = c < n1;
          const T* col = R + (ok ? c : 0);
#pragma unroll
          for (int j = 0; j < G - 1; ++j) a[u][j] = ok ? col[(int64_t)(g0 + j) * n1] : ident;
#pragma unroll
          for (int j = 0; j < G - 1; ++j)
            bq[u][j] = ok && mid_e + j < n0 ? col[(int64_t)(mid_e + j) * n1] : ident;
          mv[u] = ident;
        }
        for (int y0 = mid_s; y0 < mid_e; y0 += MB) {
          T q[CW][MB];
#pragma unroll
          for (int u = 0; u < CW; ++u) {
            const int c = cb + u * blockDim.x;
#pragma unroll
            for (int j = 0; j < MB; ++j)
              q[u][j] = (c < n1 && y0 + j < mid_e) ? R[(int64_t)(y0 + j) * n1 + c] : ident;
          }
#pragma unroll
          for (int u = 0; u < CW; ++u)
#pragma unroll
            for (int j = 0; j < MB; ++j) mv[u] = Op::apply(mv[u], q[u][j]);
        }
#pragma unroll
        for (int u = 0; u < CW; ++u) {
          const int c = cb + u * blockDim.x;
          if (c >= n1) continue;
          // A_j: suffix over in-group rows j..G-2; B_j: prefix over the G-1 rows past the middle
          T w[G];
          T run = mv[u];
          w[G - 1] = mv[u];
#pragma unroll
          for (int j = G - 2; j >= 0; --j) {
            run = Op::apply(a[u][j], run);
            w[j] = run;
          }
          T bp = ident;
#pragma unroll
          for (int j = 1; j < G; ++j) {
            bp = Op::apply(bp, bq[u][j - 1]);  // rows [mid_e, mid_e + j) (identity past n0)
            w[j] = Op::apply(w[j], bp);
          }
          const int po = poff<C>(c);
#pragma unroll
          for (int j = 0; j < G; ++j) Wt[j][po] = w[j];
        }
      }
    } else {
      // a short last group or k0 < G: each row's window directly
      for (int c = threadIdx.x; c < n1; c += blockDim.x) {
        const int po = poff<C>(c);
        for (int j = 0; j < gm; ++j) {
          const int x0 = g0 + j;
          const int e = x0 + k0 < n0 ? x0 + k0 : n0;
          T v = ident;
          for (int y = x0; y < e; ++y) v = Op::apply(v, R[(int64_t)y * n1 + c]);
          Wt[j][po] = v;
        }
      }
    }
    __syncthreads();
    // ---- row round: warp per row ----
    if (warp < gm) {
      T* wr = &Wt[warp][lane * (C + 1)];
      T* sr = &Sr[warp][0];
      const int xc = lane * C;
      T av[C];
      T lt = ident;
#pragma unroll
      for (int j = 0; j < C; ++j) {
        av[j] = xc + j < n1 ? wr[j] : ident;
        lt = Op::apply(lt, av[j]);
      }
      T pin = lt, sin = lt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const T tp = __shfl_up_sync(0xffffffffu, pin, d);
        const T ts = __shfl_down_sync(0xffffffffu, sin, d);
        if (lane >= d) pin = Op::apply(tp, pin);
        if (lane + d < 32) sin = Op::apply(sin, ts);
      }
      T pe = __shfl_up_sync(0xffffffffu, pin, 1);
      T run = __shfl_down_sync(0xffffffffu, sin, 1);
      if (lane == 0) pe = ident;
      if (lane == 31) run = ident;
      T* sl = sr + lane * (C + 1);
#pragma unroll
      for (int j = C - 1; j >= 0; --j) {
        run = Op::apply(av[j], run);
        sl[j] = run;
      }
      __syncwarp();
      const T tail = t1[warp];
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const int y = xc + j + k1;
        const T sv = y < n1 ? sr[poff<C>(y)] : ident;
        const T o = Op::apply(Op::apply(pe, sv), tail);  // P[x-1] (+) S[x+k1] (+) T1
        pe = Op::apply(pe, av[j]);
        wr[j] = o;
      }
      __syncwarp();
      T* orow = Tout + (int64_t)(g0 + warp) * n1;
      for (int x = lane; x < n1; x += 32) orow[x] = Wt[warp][poff<C>(x)];
    }
    __syncthreads();  // Wt / t1 / sh are rewritten by the next group
  }
}

int tail_chunk(int64_t n1) {
  return n1 <= 32 ? 1 : n1 <= 64 ? 2 : n1 <= 128 ? 4 : n1 <= 256 ? 8 : n1 <= 512 ? 16 : n1 <= 1024 ? 32 : 0;
}

template <class T, class Op, int C>
int go_group_c(const void* R, const void* R2, void* Tout, int64_t n0, int64_t n1, int64_t k0,
               int64_t k1, int64_t gb, int64_t ge, cudaStream_t s);

template <class T, class Op, int C>
int go_tail_c(const void* part, int64_t ppr, void* R, void* R2, void* Tout, int64_t n0, int64_t n1,
              int64_t k0, int64_t k1, cudaStream_t s, int stage) {
  if (stage == 0) {
    int64_t g1 = n0;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (g1 > cap) g1 = cap;
    k_tail_rows<T, Op><<<(unsigned)g1, kTailThreads, 0, s>>>((const T*)part, ppr, (T*)R, (T*)R2, n0, n1);
    return 1;
  }
  return go_group_c<T, Op, C>(R, R2, Tout, n0, n1, k0, k1, 0, n0, s);
}

template <class T, class Op, int C>
int go_group_c(const void* R, const void* R2, void* Tout, int64_t n0, int64_t n1, int64_t k0,
               int64_t k1, int64_t gb, int64_t ge, cudaStream_t s) {
  int64_t g2 = (ge - gb + kGroup - 1) / kGroup;
  const int64_t cap2 = (int64_t)num_sms() * 16;
  if (g2 > cap2) g2 = cap2;
  if (g2 < 1) return 0;
  k_tail_group<T, Op, C><<<(unsigned)g2, kGroupThreads, 0, s>>>((const T*)R, (const T*)R2, (T*)Tout,
                                                                (int)n0, (int)n1, (int)k0, (int)k1,
                                                                (int)gb, (int)ge);
  return 1;
}

template <class T, class Op>
int go_tail(const void* part, int64_t ppr, void* R, void* R2, void* Tout, int64_t n0, int64_t n1,
            int64_t k0, int64_t k1, cudaStream_t s, int stage) {
  switch (tail_chunk(n1)) {
    case 1: return go_tail_c<T, Op, 1>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
    case 2: return go_tail_c<T, Op, 2>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
    case 4: return go_tail_c<T, Op, 4>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
    case 8: return go_tail_c<T, Op, 8>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
    case 16: return go_tail_c<T, Op, 16>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
    case 32:
      if constexpr (sizeof(T) == 4) return go_tail_c<T, Op, 32>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
      return -1;
  }
  return -1;
}

// A shard of the tail: stage 0 R2[i] = fold of R row i (n_rows rows of R);
// stage 1 T rows [gb, ge) with R and Tout indexed by the global row.
template <class T, class Op>
int go_tail_shard(const void* R, void* R2, void* Tout, int64_t n0, int64_t n1, int64_t k0,
                  int64_t k1, int64_t gb, int64_t ge, cudaStream_t s, int stage) {
  if (stage == 0) {
    const int64_t rows = ge - gb;
    if (rows <= 0) return 0;
    int64_t g1 = rows;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (g1 > cap) g1 = cap;
    k_tail_rows<T, Op><<<(unsigned)g1, kTailThreads, 0, s>>>(nullptr, 0, (T*)R, (T*)R2, rows, n1);
    return 1;
  }
  switch (tail_chunk(n1)) {
    case 1: return go_group_c<T, Op, 1>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s);
    case 2: return go_group_c<T, Op, 2>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s);
    case 4: return go_group_c<T, Op, 4>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s);
    case 8: return go_group_c<T, Op, 8>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s);
    case 16: return go_group_c<T, Op, 16>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s);
    case 32:
      if constexpr (sizeof(T) == 4) return go_group_c<T, Op, 32>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s);
      return -1;
  }
  return -1;
}

}  // namespace

int launch_tail2d_shard(int dtype, int op, const void* R, void* R2, void* Tout, int64_t n0,
                        int64_t n1, int64_t k0, int64_t k1, int64_t gb, int64_t ge, cudaStream_t s,
                        int stage) {
  if (dtype == F32 && op == ADD) return go_tail_shard<float, OpAdd>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s, stage);
  if (dtype == F64 && op == ADD) return go_tail_shard<double, OpAdd>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s, stage);
  if (dtype == I64 && op == ADD) return go_tail_shard<i64, OpAdd>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s, stage);
  if (dtype == I64 && op == MAX) return go_tail_shard<i64, OpMax>(R, R2, Tout, n0, n1, k0, k1, gb, ge, s, stage);
  return -2;
}

int tail2d_ok(int dtype, int64_t n0, int64_t n1, int64_t k0) {
  const char* e = getenv("EXSUM_TAIL2D");  // 0: the recursive tail (measurement)
  if (e && e[0] == '0') return 0;
  // static shared rows: 2 G rows of 32 (C + 1) elements (<= 2 * 4 * 33 * 32 * 8 B = 66 KB
  // would exceed the 48 KB static limit for 8-byte rows of 1024: those take the old path)
  const int C = tail_chunk(n1);
  if (!C || n0 > (1 << 30) || k0 < 1) return 0;
  return (size_t)2 * kGroup * 32 * (C + 1) * dtype_size(dtype) <= 46 * 1024 ? 1 : 0;
}

int launch_tail2d(int dtype, int op, const void* part, int64_t ppr, void* R, void* R2, void* Tout,
                  int64_t n0, int64_t n1, int64_t k0, int64_t k1, cudaStream_t s, int stage) {
  if (dtype == F32 && op == ADD) return go_tail<float, OpAdd>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
  if (dtype == F64 && op == ADD) return go_tail<double, OpAdd>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
  if (dtype == I64 && op == ADD) return go_tail<i64, OpAdd>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
  if (dtype == I64 && op == MAX) return go_tail<i64, OpMax>(part, ppr, R, R2, Tout, n0, n1, k0, k1, s, stage);
  return -2;
}

}  // namespace exsum
