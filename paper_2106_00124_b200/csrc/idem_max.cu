// idem_max.cu -- box-complement (strong excluded sum) for an idempotent
// operator (max) as per-axis marginals: two HBM passes in total.
//
// The reference's box_complement_excluded (excluded.py:129-159) covers the
// complement of the box B(x) = prod_a [x_a, x_a + k_a) by disjoint slabs.  For
// an idempotent monoid the slabs may overlap, and the complement is the union
// of the 2d half-space slabs {y : y_a < x_a} and {y : y_a >= x_a + k_a}.  Each
// of those is a full fold over every axis but a, so with the marginals
//   M_a[i] = (+)_{y : y_a = i} A[y]                      (fold over all axes but a)
//   F_a[i] = P_a[i - 1] (+) S_a[i + k_a]                  (1-D excluded window of M_a;
//                                                          P / S inclusive prefix /
//                                                          suffix, out of range = identity)
// the excluded sum is
//   out[x] = F_0[x_0] (+) F_1[x_1] (+) ... (+) F_{d-1}[x_{d-1}]
// -- every term a fold of elements of x's complement, every element of the
// complement in at least one term, no inverse anywhere: for max the result is
// bit-identical to the slab algorithm's (max is exact).  An empty complement
// (k_a = n_a on every axis) leaves the identity, as in the reference.
//
// Launches:
//   k_idem_scan   one read of A (after a memset of the marginal images): a warp
//                 per (16 rows, strip of up to 512 columns), 16-byte streaming
//                 loads one row ahead; per row a warp fold, combined over lanes
//                 with equal leading coordinates (segmented warp fold) and
//                 atomically max'ed into M_a (a < d-1); per column the fold over
//                 the CTA's rows, atomically into M_{d-1};
//   k_idem_bcast  one write of out: a grid of 2 CTAs per SM; every CTA first
//                 builds F (a warp per axis: chunk folds, warp scans for the
//                 carries, suffix stage, then P[i-1] (+) S[i+k]) from the
//                 marginals in shared memory, then its warps take units of 4
//                 rows in turn: per row the fold of the leading F_a and
//                 out = that (+) F_{d-1}[column] -- 16-byte streaming stores.
// DRAM traffic 2 N s against 4 N s for the slab route (C2 box-complement max
// 0.127 -> 0.055 ms; a plain read of the same 134 MB takes 29-31 us and a plain
// write 25-27 us on B200, tools/bw_probe.cu); a read-all-then-write-all schedule is the floor for any
// excluded sum (every output depends on the whole input).
#include <stdlib.h>

#include <algorithm>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

namespace {

#ifndef IDEM_THREADS
#define IDEM_THREADS 256
#endif
constexpr int kIdemThreads = IDEM_THREADS;
constexpr int kIdemWarps = kIdemThreads / 32;
#ifndef IDEM_RBU
#define IDEM_RBU 16
#endif
#ifndef IDEM_UR
#define IDEM_UR 1
#endif
#ifndef IDEM_MINB
#define IDEM_MINB 4
#endif
constexpr int kRbu = IDEM_RBU;  // rows per warp work unit (<= 32: lane l keeps row l's fold)
constexpr int kIdemMaxSum = 4096;  // sum of the extents: every broadcast CTA stages 2 S of tables

struct IdemShape {
  int d;
  int64_t ext[EXSUM_IDEM_MAX_DIMS];
  int64_t k[EXSUM_IDEM_MAX_DIMS];
  int64_t off[EXSUM_IDEM_MAX_DIMS];  // table offset of axis a (sum of the extents before it)
  int64_t rows, nl;                  // rows held here (a shard: its own), nl = n_{d-1}
  int64_t S;                         // sum of the extents
  int64_t row_off;                   // global index of the first row held here (a shard's)
};

// The marginals accumulate with atomic max on the order-preserving unsigned
// image of the value (sign bit flipped): the identity INT64_MIN maps to 0, so a
// byte memset initialises them.
__device__ __forceinline__ unsigned long long bias(i64 v) {
  return (unsigned long long)v ^ 0x8000000000000000ULL;
}
__device__ __forceinline__ i64 unbias(unsigned long long u) {
  return (i64)(u ^ 0x8000000000000000ULL);
}

// Work units: (block of kRbu rows, strip of W = 32 * VE * NV columns), a warp
// each; a CTA's 8 warps take 8 consecutive row blocks of one strip.
struct IdemTiling {
  int VE, NV, W;
  int64_t nstrip, nrb, ncta;
};
IdemTiling idem_tiling(const IdemShape& s, bool vec) {
  IdemTiling t;
  t.VE = vec ? 2 : 1;
  const int64_t ncv = (s.nl + t.VE - 1) / t.VE;
  int nv = 1;
  while (nv < 8 && 32 * nv < ncv) nv <<= 1;
  t.NV = nv;
  t.W = 32 * t.VE * nv;
  t.nstrip = (s.nl + t.W - 1) / t.W;
  t.nrb = (s.rows + kRbu - 1) / kRbu;
  t.ncta = t.nstrip * ((t.nrb + kIdemWarps - 1) / kIdemWarps);
  return t;
}

// A warp's rows: lane l owns NV vectors of every row (vector q at column
// lane * VE + q * 32 VE), folds them into its column accumulators and, by a
// warp reduction, each row into rmax of lane (row index).  FULL: 32 rows and
// the whole strip in range -- unpredicated loads, so all UR * NV of them are in
// flight at once (a predicated identity fill of a load's register waits for
// that load and serialises the batch).
template <class T, class Op, int VE, int NV, bool FULL>
__device__ __forceinline__ void idem_rows(const T* __restrict__ src, int64_t nl, int nr, int lane,
                                          T (&cacc)[NV][VE], T& rmax, int64_t cols = 0) {
  typedef Vec<T, VE> VT;
  const T ident = Op::template identity<T>();
  constexpr int UR = IDEM_UR;  // rows per stage
  auto fold = [&](const VT (&v)[UR][NV], int i0) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      T rm = ident;
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int j = 0; j < VE; ++j) {
          cacc[q][j] = Op::apply(cacc[q][j], v[u][q].v[j]);
          rm = Op::apply(rm, v[u][q].v[j]);
        }
#pragma unroll
      for (int dd = 16; dd >= 1; dd >>= 1) rm = Op::apply(rm, __shfl_xor_sync(0xffffffffu, rm, dd));
      if (lane == i0 + u) rmax = rm;
    }
  };
  if constexpr (FULL) {
    // kRbu rows in stages of UR, the next stage's loads issued before the
    // current stage is folded (two stages in flight)
    constexpr int NS = kRbu / UR;
    VT buf[2][UR][NV];
    auto load = [&](VT (&v)[UR][NV], int i0) {
#pragma unroll
      for (int u = 0; u < UR; ++u)
#pragma unroll
        for (int q = 0; q < NV; ++q)
          v[u][q] = ld_stream<T, VE>(src + (int64_t)(i0 + u) * nl + q * 32 * VE);
    };
    load(buf[0], 0);
#pragma unroll
    for (int st = 0; st < NS; ++st) {
      if (st + 1 < NS) load(buf[(st + 1) & 1], (st + 1) * UR);
      fold(buf[st & 1], st * UR);
    }
  } else {
    for (int i0 = 0; i0 < nr; i0 += UR) {
      VT v[UR][NV];
#pragma unroll
      for (int u = 0; u < UR; ++u)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const bool ok = i0 + u < nr && lane * VE + q * 32 * VE < cols;
          const int64_t o = ok ? (int64_t)(i0 + u) * nl + q * 32 * VE : 0;
          v[u][q] = ld_stream<T, VE>(src - lane * VE * (ok ? 0 : 1) + o);  // a valid address either way
          if (!ok) {
#pragma unroll
            for (int j = 0; j < VE; ++j) v[u][q].v[j] = ident;
          }
        }
      fold(v, i0);
    }
  }
}

// One read of A: per row the fold (warp reduce) into the leading marginals,
// per column the fold over the CTA's rows into the last-axis marginal (atomic
// max on the biased image).
template <class T, class Op, int VE, int NV>
__global__ void __launch_bounds__(kIdemThreads, (NV >= 8 ? 2 : IDEM_MINB) * 256 / kIdemThreads)
k_idem_scan(const T* __restrict__ in, unsigned long long* __restrict__ Mu, IdemShape s,
            int64_t nstrip, int64_t nrb) {
  typedef Vec<T, VE> VT;
  constexpr int W = 32 * VE * NV;
  __shared__ T csh[kIdemWarps][W];
  const T ident = Op::template identity<T>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t strip = blockIdx.x % nstrip;
  const int64_t rb = (blockIdx.x / nstrip) * kIdemWarps + warp;
  const int64_t c0 = strip * W;
  T cacc[NV][VE];
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int j = 0; j < VE; ++j) cacc[q][j] = ident;
  if (rb < nrb) {
    const int64_t r0 = rb * kRbu;
    const int nr = (int)min((int64_t)kRbu, s.rows - r0);
    const T* src = in + r0 * s.nl + c0 + lane * VE;
    T rmax = ident;  // lane l: the fold of row r0 + l
    if (nr == kRbu && c0 + W <= s.nl) {
      idem_rows<T, Op, VE, NV, true>(src, s.nl, kRbu, lane, cacc, rmax);
    } else {
      idem_rows<T, Op, VE, NV, false>(src, s.nl, nr, lane, cacc, rmax, s.nl - c0);
    }
    // the warp's 32 consecutive rows into the leading marginals: per axis a,
    // rows with equal r / stride_a form contiguous lane segments; a segmented
    // suffix fold leaves each segment's fold in its first lane, which issues
    // one atomic (C2 axis 0: one atomic per warp instead of 32 on one address)
    int64_t key = s.row_off + r0 + lane;  // global row / stride_a, axis by axis from the last
    for (int a = s.d - 2; a >= 0; --a) {
      T v = lane < nr ? rmax : ident;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const T ov = __shfl_down_sync(0xffffffffu, v, dd);
        const int64_t ok = __shfl_down_sync(0xffffffffu, key, dd);
        if (lane + dd < 32 && ok == key) v = Op::apply(v, ov);
      }
      const int64_t pk = __shfl_up_sync(0xffffffffu, key, 1);
      const int64_t q = key / s.ext[a];
      if (lane < nr && (lane == 0 || pk != key)) atomicMax(Mu + s.off[a] + (key - q * s.ext[a]), bias(v));
      key = q;
    }
  }
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int j = 0; j < VE; ++j) csh[warp][q * 32 * VE + lane * VE + j] = cacc[q][j];
  __syncthreads();
  for (int c = tid; c < W; c += kIdemThreads) {
    if (c0 + c >= s.nl) continue;
    T m = csh[0][c];
#pragma unroll
    for (int w = 1; w < kIdemWarps; ++w) m = Op::apply(m, csh[w][c]);
    atomicMax(Mu + s.off[s.d - 1] + c0 + c, bias(m));
  }
}

template <class T, class Op, int VE, int NV, int RB>
__device__ __forceinline__ void idem_bcast_unit(const T* F, T* __restrict__ out, const IdemShape& s,
                                                int64_t strip, int64_t rb, int lane);

// The broadcast's grid: IDEM_BGRID CTAs per SM (0: one CTA per 8 row
// blocks of the scan's tiling) over warp units of IDEM_BRB rows.  C2 (256^3):
// 2 / 4 -> broadcast 33.1 -> 29.1 us (0/16 leaves the SMs 3-4 CTAs each, and
// every CTA builds the tables; 1-2 per SM with 4-row units balance to ~1%).
#ifndef IDEM_BGRID
#define IDEM_BGRID 2
#endif
#ifndef IDEM_BRB
#define IDEM_BRB 4
#endif

// One write of out.  Prologue (every CTA, redundantly -- the tables are at
// most kIdemMaxSum elements): the marginals from Mu into shared memory, then a
// warp per axis builds F_a in place: lane chunks, warp scans of the chunk
// folds for the carries, the inclusive suffix into a second stage, then
// F[i] = P[i-1] (+) S[i+k_a] (out-of-range terms the identity).  Then lane l
// folds the leading F terms of row r0 + l and the warp walks its rows with
// out = that (+) F_{d-1}[column].
template <class T, class Op, int VE, int NV>
__global__ void __launch_bounds__(kIdemThreads)
k_idem_bcast(const unsigned long long* __restrict__ Mu, T* __restrict__ out, IdemShape s,
             int64_t nstrip, int64_t nrb, unsigned long long flip) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* F = reinterpret_cast<T*>(smem);  // [S]: M, then F
  T* Ss = F + s.S;                    // [S]: inclusive suffixes
  const T ident = Op::template identity<T>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the marginals: biased images (flip = sign bit) or, for a shard, plain values (flip = 0)
  for (int64_t i = tid; i < s.S; i += kIdemThreads) F[i] = (T)(Mu[i] ^ flip);
  __syncthreads();
  for (int a = warp; a < s.d; a += kIdemWarps) {
    const int n = (int)s.ext[a];
    T* m = F + s.off[a];
    T* sx = Ss + s.off[a];
    const int L = (n + 31) / 32;
    const int lo = min(n, lane * L), hi = min(n, lo + L);
    T tot = ident;
    for (int i = lo; i < hi; ++i) tot = Op::apply(tot, m[i]);
    T pin = tot, sin = tot;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const T tp = __shfl_up_sync(0xffffffffu, pin, dd);
      const T ts = __shfl_down_sync(0xffffffffu, sin, dd);
      if (lane >= dd) pin = Op::apply(tp, pin);
      if (lane + dd < 32) sin = Op::apply(sin, ts);
    }
    T pre = __shfl_up_sync(0xffffffffu, pin, 1);   // fold of the chunks before
    T run = __shfl_down_sync(0xffffffffu, sin, 1);  // fold of the chunks after
    if (lane == 0) pre = ident;
    if (lane == 31) run = ident;
    for (int i = hi - 1; i >= lo; --i) {
      run = Op::apply(m[i], run);
      sx[i] = run;  // S[i]
    }
    __syncwarp();
    const int64_t k = s.k[a];
    for (int i = lo; i < hi; ++i) {
      const T mi = m[i];
      m[i] = i + k < n ? Op::apply(pre, sx[i + k]) : pre;  // P[i-1] (+) S[i+k]
      pre = Op::apply(pre, mi);
    }
  }
  __syncthreads();
#if IDEM_BGRID
  // a grid of IDEM_BGRID CTAs per SM: warp units (row block, strip) taken in
  // turn, the tables built once per CTA
  const int64_t nrb_b = (s.rows + IDEM_BRB - 1) / IDEM_BRB;
  for (int64_t u = (int64_t)blockIdx.x * kIdemWarps + warp; u < nrb_b * nstrip;
       u += (int64_t)gridDim.x * kIdemWarps) {
    idem_bcast_unit<T, Op, VE, NV, IDEM_BRB>(F, out, s, u % nstrip, u / nstrip, lane);
  }
#else
  const int64_t strip = blockIdx.x % nstrip;
  const int64_t rb = (blockIdx.x / nstrip) * kIdemWarps + warp;
  if (rb >= nrb) return;
  idem_bcast_unit<T, Op, VE, NV, kRbu>(F, out, s, strip, rb, lane);
#endif
}

template <class T, class Op, int VE, int NV, int RB>
__device__ __forceinline__ void idem_bcast_unit(const T* F, T* __restrict__ out, const IdemShape& s,
                                                int64_t strip, int64_t rb, int lane) {
  typedef Vec<T, VE> VT;
  constexpr int W = 32 * VE * NV;
  const T ident = Op::template identity<T>();
  const int64_t c0 = strip * W;
  const int64_t r0 = rb * RB;
  const int nr = (int)min((int64_t)RB, s.rows - r0);
  T crow = ident;
  if (lane < nr) {
    int64_t r = s.row_off + r0 + lane;
    for (int a = s.d - 2; a >= 0; --a) {
      const int64_t q = r / s.ext[a];
      crow = Op::apply(crow, F[s.off[a] + (r - q * s.ext[a])]);
      r = q;
    }
  }
  T fc[NV][VE];
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int j = 0; j < VE; ++j) {
      const int64_t c = c0 + lane * VE + q * 32 * VE + j;
      fc[q][j] = c < s.nl ? F[s.off[s.d - 1] + c] : ident;
    }
  T* dst = out + r0 * s.nl + c0 + lane * VE;
  for (int i = 0; i < nr; ++i) {
    const T c = __shfl_sync(0xffffffffu, crow, i);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      if (c0 + lane * VE + q * 32 * VE < s.nl) {
        VT v;
#pragma unroll
        for (int j = 0; j < VE; ++j) v.v[j] = Op::apply(c, fc[q][j]);
        st_stream<T, VE>(dst + (int64_t)i * s.nl + q * 32 * VE, v);
      }
    }
  }
}

// stage -1: workspace bytes only; 0: memset + scan, 1: broadcast (with the tables)
template <class T, class Op, int VE, int NV>
void launch_stage(const T* in, T* out, const IdemShape& s, const IdemTiling& t,
                  unsigned long long* Mu, cudaStream_t st, int stage, unsigned long long flip) {
  const unsigned grid = (unsigned)t.ncta;
  if (stage == 0) {
    k_idem_scan<T, Op, VE, NV><<<grid, kIdemThreads, 0, st>>>(in, Mu, s, t.nstrip, t.nrb);
  } else {
    const size_t sm = (size_t)2 * s.S * sizeof(T);
    ensure_smem((const void*)k_idem_bcast<T, Op, VE, NV>, sm);
    unsigned bgrid = grid;
#if IDEM_BGRID
    bgrid = (unsigned)std::min<int64_t>(grid, (int64_t)num_sms() * IDEM_BGRID);
#endif
    k_idem_bcast<T, Op, VE, NV><<<bgrid, kIdemThreads, sm, st>>>(Mu, out, s, t.nstrip, t.nrb, flip);
  }
}

// stage 2 (a shard): the broadcast from plain marginals `marg` (the all-reduced
// global ones) instead of the workspace's biased images
template <class T, class Op>
int go_idem(const T* in, T* out, const IdemShape& s, void* ws, cudaStream_t st, int stage,
            size_t* bytes, const void* marg = nullptr) {
  const bool vec = s.nl % 2 == 0 && ((uintptr_t)in % 16) == 0 && ((uintptr_t)out % 16) == 0 &&
                   sizeof(T) == 8;
  const IdemTiling t = idem_tiling(s, vec);
  // workspace: Mu [S], the marginals' biased images
  if (bytes) *bytes = (size_t)s.S * 8;
  if (stage < 0) return 0;
  unsigned long long* Mu = stage == 2 ? (unsigned long long*)marg : static_cast<unsigned long long*>(ws);
  const unsigned long long flip = stage == 2 ? 0ULL : 0x8000000000000000ULL;
  if (stage == 2) stage = 1;
  // the marginals start at zero (= the identity's image)
  if (stage == 0 && cudaMemsetAsync(Mu, 0, (size_t)s.S * 8, st) != cudaSuccess) return -1;
#define IDEM_GO(VE_, NV_) launch_stage<T, Op, VE_, NV_>(in, out, s, t, Mu, st, stage, flip)
  if (t.VE == 2) {
    switch (t.NV) {
      case 1: IDEM_GO(2, 1); break;
      case 2: IDEM_GO(2, 2); break;
      case 4: IDEM_GO(2, 4); break;
      default: IDEM_GO(2, 8); break;
    }
  } else {
    switch (t.NV) {
      case 1: IDEM_GO(1, 1); break;
      case 2: IDEM_GO(1, 2); break;
      case 4: IDEM_GO(1, 4); break;
      default: IDEM_GO(1, 8); break;
    }
  }
#undef IDEM_GO
  return 1;
}

__global__ void k_idem_unbias(const unsigned long long* __restrict__ Mu, i64* __restrict__ marg,
                              int64_t S) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S;
       i += (int64_t)gridDim.x * blockDim.x)
    marg[i] = unbias(Mu[i]);
}

}  // namespace

int idem_max_ok(int dtype, int op, int d, const int64_t* ext) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("EXSUM_IDEM");  // 0: the slab route for max too (measurement)
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (!env || op != MAX || dtype != I64) return 0;
  if (d < 2 || d > EXSUM_IDEM_MAX_DIMS) return 0;
  int64_t S = 0;
  for (int a = 0; a < d; ++a) S += ext[a];
  return S <= kIdemMaxSum ? 1 : 0;
}

// A shard of the global array: `in` / `out` hold global planes [x0, x0 + n_own)
// of axis 0.  stage 0: the shard's marginals as plain values into `marg`
// (S = sum of the global extents; the identity where the shard has no
// element), through the biased images in `ws`; stage 1: the shard's output
// planes from the all-reduced global marginals `marg`.
int launch_idem_max_shard(int dtype, const void* in, void* out, void* marg, int d,
                          const int64_t* ext, const int64_t* k, int64_t x0, int64_t n_own,
                          void* ws, size_t* ws_bytes, cudaStream_t st, int stage) {
  if (dtype != I64) return -1;
  IdemShape s;
  s.d = d;
  s.S = 0;
  int64_t per_plane = 1;
  for (int a = 0; a < d; ++a) {
    s.ext[a] = ext[a];
    s.k[a] = k[a];
    s.off[a] = s.S;
    s.S += ext[a];
    if (a > 0) per_plane *= ext[a];
  }
  s.nl = ext[d - 1];
  const int64_t rows_per_plane = per_plane / s.nl;
  s.rows = n_own * rows_per_plane;
  s.row_off = x0 * rows_per_plane;
  if (stage < 0 || s.rows == 0) {
    if (ws_bytes) *ws_bytes = (size_t)s.S * 8;
    if (stage >= 0 && s.rows == 0 && stage == 0) {
      // no planes here: every marginal entry is the identity
      if (cudaMemsetAsync(ws, 0, (size_t)s.S * 8, st) != cudaSuccess) return -1;
      k_idem_unbias<<<(unsigned)((s.S + 255) / 256), 256, 0, st>>>(
          static_cast<const unsigned long long*>(ws), static_cast<i64*>(marg), s.S);
      return 1;
    }
    return 0;
  }
  if (stage == 0) {
    int rc = go_idem<i64, OpMax>(static_cast<const i64*>(in), nullptr, s, ws, st, 0, ws_bytes);
    if (rc < 0) return rc;
    k_idem_unbias<<<(unsigned)((s.S + 255) / 256), 256, 0, st>>>(
        static_cast<const unsigned long long*>(ws), static_cast<i64*>(marg), s.S);
    return rc + 1;
  }
  return go_idem<i64, OpMax>(nullptr, static_cast<i64*>(out), s, nullptr, st, 2, ws_bytes, marg);
}

int launch_idem_max(int dtype, const void* in, void* out, int d, const int64_t* ext,
                    const int64_t* k, void* ws, size_t* ws_bytes, cudaStream_t st, int stage) {
  if (dtype != I64) return -1;
  IdemShape s;
  s.d = d;
  s.S = 0;
  int64_t N = 1;
  for (int a = 0; a < d; ++a) {
    s.ext[a] = ext[a];
    s.k[a] = k[a];
    s.off[a] = s.S;
    s.S += ext[a];
    N *= ext[a];
  }
  s.nl = ext[d - 1];
  s.rows = N / s.nl;
  s.row_off = 0;
  return go_idem<i64, OpMax>(static_cast<const i64*>(in), static_cast<i64*>(out), s, ws, st, stage,
                             ws_bytes);
}

}  // namespace exsum
