// tile_pair.cu -- the last two windowed passes of BDBS in one launch for
// windows the fused pass pair has no template for (k = 32, or rows that are
// not 256/512/1024 wide): C1 (2-D float64 1024^2, box 32^2) and the 32^3 box
// of C5.
//
// Same algorithm and association as windowed_sum_axis (scan.py:61-102) applied
// along axis d-2 and then along axis d-1 (included.py:124-129): in-block
// right-nested suffix, left-nested prefix of the next block, one stitch
// combine -- float results are bit-identical to the reference's.
//
// B200 mapping: a CTA owns an output tile of K rows (one K-block of axis d-2)
// x TW = 4K columns (whole K-blocks of axis d-1) of one outer index:
//   * column pass: a thread per column of the tile plus its K-column halo (the
//     row pass's stitch partner), the block's K values and the next block's
//     rows loaded straight from global into registers (lanes on consecutive
//     columns: coalesced, all loads of a column in flight at once), suffix,
//     prefix and stitch in registers, the K results into a shared stage;
//   * row pass: a thread per (row, K-block), lanes on consecutive rows of the
//     stage (odd row pitch: conflict-free): phase A writes the left-nested
//     prefixes of the stitch-partner blocks to a second stage, phase B runs
//     the in-block suffix in place and stitches;
//   * the tile leaves as coalesced streaming stores (with the BDBSC
//     complement epilogue when `total` is given).
// The next-block rows and halo columns are re-read from L2 by the
// neighbouring tiles; the input is read from HBM once: 2 N s of DRAM traffic
// for both passes instead of 4 N s, and one launch instead of two.
#include <stdlib.h>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

#ifndef TILE_TWB
#define TILE_TWB 4
#endif
#ifndef TILE_MINB
#define TILE_MINB 2
#endif

// One tile of K output rows x TW output columns; the stage t holds the input
// tile's 2K rows x (TW + K) columns at an odd row pitch P (lanes on rows:
// conflict-free scalar accesses), filled by element-granular cp.async (a warp
// per row, coalesced).  The column pass runs in place on the K output rows
// (the next block's rows K..2K-1 are only read), then the row pass in two
// phases: A writes the left-nested prefixes of the stitch-partner blocks into
// the dead rows K..2K-1, B runs the in-block suffix in place and stitches.
// Geometry is compile-time (TW = TILE_TWB K, P = (TW + K) | 1), so every
// shared-memory offset of the chains is an immediate; FULL (an interior tile:
// 2K rows and TW + K columns in range) drops every bound check.
template <class T, class Op, int K, bool FULL>
__device__ __forceinline__ void tile_body(T* t, const T* __restrict__ src, T* __restrict__ dst,
                                          int64_t n2, int rows_in, int cols_in, int rows_out,
                                          int cols_out, int nlen1, int64_t ncols_after, bool epi,
                                          T tot) {
  constexpr int TW = TILE_TWB * K, TC = TW + K, P = TC | 1, NBC = TW / K;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (FULL) {
    rows_in = 2 * K;
    cols_in = TC;
    rows_out = K;
    cols_out = TW;
    nlen1 = K;
  }
  for (int r = tid >> 5; r < rows_in; r += blockDim.x >> 5)
    for (int c = lane; c < cols_in; c += 32)
      cp_async_n<sizeof(T)>(t + r * P + c, src + (int64_t)r * n2 + c);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // ---- column pass (axis d-2), in place: a thread per column ----
  for (int cc = tid; cc < cols_in; cc += blockDim.x) {
    T* col = t + cc;
    const int blen = rows_out;
    T sv = col[(blen - 1) * P];
#pragma unroll
    for (int r = K - 2; r >= 0; --r)
      if (FULL || r < blen - 1) {
        sv = Op::apply(col[r * P], sv);
        col[r * P] = sv;
      }
    if (FULL || nlen1 > 0) {
      T Pr = col[K * P];
#pragma unroll
      for (int r = 1; r < K; ++r) {
        const int jj = r - 1;
        if (jj >= 1 && (FULL || jj < nlen1)) Pr = Op::apply(Pr, col[(K + jj) * P]);
        col[r * P] = Op::apply(col[r * P], Pr);
      }
    }
  }
  __syncthreads();

  // ---- row pass (axis d-1): a thread per (row, block), lanes on rows ----
  const int r = lane;
  const int j = tid >> 5;
  for (int jb = j; jb <= NBC; jb += blockDim.x >> 5) {  // phase A: prefixes of blocks 1..NBC
    if ((FULL || r < rows_out) && jb >= 1 && (FULL || jb * K < cols_in)) {
      const T* w = t + r * P + jb * K;
      T* pb = t + (K + r) * P + jb * K;
      const int plen = FULL ? K - 1 : min(K - 1, cols_in - jb * K);
      T Pr = w[0];
      pb[0] = Pr;
#pragma unroll
      for (int q = 1; q < K - 1; ++q)
        if (FULL || q < plen) {
          Pr = Op::apply(Pr, w[q]);
          pb[q] = Pr;
        }
    }
  }
  __syncthreads();
  for (int jb = j; jb < NBC; jb += blockDim.x >> 5) {  // phase B
    if ((FULL || r < rows_out) && (FULL || jb * K < cols_out)) {
      T* w = t + r * P + jb * K;
      const T* pn = t + (K + r) * P + (jb + 1) * K;
      // columns of this block and of the next one (tile columns past this block)
      const int64_t rem = FULL ? 2 * K : ncols_after - jb * K;
      const int blen = (int)(rem < K ? rem : K);
      T sv = w[blen - 1];
#pragma unroll
      for (int q = K - 2; q >= 0; --q)
        if (FULL || q < blen - 1) {
          sv = Op::apply(w[q], sv);
          w[q] = sv;
        }
      if (FULL || rem > K) {
        const int nlen = FULL ? K : (int)(rem - K < K ? rem - K : K);
#pragma unroll
        for (int q = 1; q < K; ++q) w[q] = Op::apply(w[q], pn[FULL ? q - 1 : min(q - 1, nlen - 1)]);
      }
    }
  }
  __syncthreads();

  // ---- store: a warp per row, coalesced ----
  for (int rr = tid >> 5; rr < rows_out; rr += blockDim.x >> 5)
    for (int c = lane; c < cols_out; c += 32) {
      const T v = t[rr * P + c];
      st1<T>(dst + (int64_t)rr * n2 + c, epi ? OpAdd::inverse<T>(tot, v) : v);
    }
  __syncthreads();  // the stage is refilled by the next tile
}

template <class T, class Op, int K>
__global__ void __launch_bounds__(256, TILE_MINB)
k_tile_pair(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n1, int64_t n2,
            const typename AccOf<T>::type* __restrict__ total) {
  constexpr int TW = TILE_TWB * K, TC = TW + K;
  extern __shared__ __align__(16) unsigned char smem[];
  T* t = reinterpret_cast<T*>(smem);  // [2K][P]
  const int64_t tiles1 = (n1 + K - 1) / K;
  const int64_t tiles2 = (n2 + TW - 1) / TW;
  const int64_t items = outer * tiles1 * tiles2;
  const bool epi = total != nullptr;
  const T tot = epi ? (T)(*total) : T(0);
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t b2 = item % tiles2;  // column tiles fastest: neighbours share halos in L2
    const int64_t rest = item / tiles2;
    const int64_t b1 = rest % tiles1;
    const int64_t o = rest / tiles1;
    const int64_t r0 = b1 * K, c0 = b2 * TW;
    const int rows_in = (int)min((int64_t)2 * K, n1 - r0);
    const int cols_in = (int)min((int64_t)TC, n2 - c0);
    const int rows_out = (int)min((int64_t)K, n1 - r0);
    const int cols_out = (int)min((int64_t)TW, n2 - c0);
    const int nlen1 = (int)max((int64_t)0, min((int64_t)K, n1 - (r0 + K)));
    const T* src = in + (o * n1 + r0) * n2 + c0;
    T* dst = out + (o * n1 + r0) * n2 + c0;
    if (rows_in == 2 * K && cols_in == TC)
      tile_body<T, Op, K, true>(t, src, dst, n2, rows_in, cols_in, rows_out, cols_out, nlen1,
                                n2 - c0, epi, tot);
    else
      tile_body<T, Op, K, false>(t, src, dst, n2, rows_in, cols_in, rows_out, cols_out, nlen1,
                                 n2 - c0, epi, tot);
  }
}

namespace {

// Tile geometry for window K: K output rows x TW = TILE_TWB K output
// columns; the stage 2K x P with P = (TW + K) | 1.
struct TileGeom {
  int TW, P;
  size_t smem;
};
TileGeom tile_geom(int K, int es) {
  TileGeom g;
  g.TW = TILE_TWB * K;
  g.P = (g.TW + K) | 1;
  g.smem = (size_t)2 * K * g.P * es;
  return g;
}

template <class T, class Op, int K>
int go_tile(const void* in, void* out, int64_t outer, int64_t n1, int64_t n2, const void* total,
            cudaStream_t s) {
  const TileGeom g = tile_geom(K, (int)sizeof(T));
  const int64_t items = outer * ((n1 + K - 1) / K) * ((n2 + g.TW - 1) / g.TW);
  int per_sm = (int)((228 * 1024) / (g.smem + 1024));
  if (per_sm > 8) per_sm = 8;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = items;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (grid > cap) grid = cap;
  auto fn = k_tile_pair<T, Op, K>;
  ensure_smem((const void*)fn, g.smem);
  fn<<<(unsigned)grid, 256, g.smem, s>>>(static_cast<const T*>(in), static_cast<T*>(out), outer, n1,
                                         n2, static_cast<const typename AccOf<T>::type*>(total));
  return 1;
}

template <class T, class Op>
int pick_tile(int64_t k, const void* in, void* out, int64_t outer, int64_t n1, int64_t n2,
              const void* total, cudaStream_t s) {
  switch (k) {
    case 32: return go_tile<T, Op, 32>(in, out, outer, n1, n2, total, s);
  }
  return -1;
}

}  // namespace

int tile_pair_ok(int dtype, int op, int64_t N, int64_t n1, int64_t n2, int64_t k1, int64_t k2) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("EXSUM_TILE_PAIR");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (!env) return 0;
  if (dtype != F32 && dtype != F64 && dtype != I64) return 0;
  if (op == MAX && dtype != I64) return 0;
  if (k1 != k2 || k1 != 32) return 0;
  if (N * (int64_t)dtype_size(dtype) > ((int64_t)64 << 20)) return 0;
  if (n1 < k1 || n2 < k2) return 0;  // clamped windows keep the single passes
  return 1;
}

int launch_tile_pair(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n1,
                     int64_t n2, int64_t k1, int64_t k2, const void* total, cudaStream_t s) {
  if (!tile_pair_ok(dtype, op, outer * n1 * n2, n1, n2, k1, k2)) return -1;
  if (dtype == F32 && op == ADD) return pick_tile<float, OpAdd>(k1, in, out, outer, n1, n2, total, s);
  if (dtype == F64 && op == ADD) return pick_tile<double, OpAdd>(k1, in, out, outer, n1, n2, total, s);
  if (dtype == I64 && op == ADD) return pick_tile<i64, OpAdd>(k1, in, out, outer, n1, n2, total, s);
  if (dtype == I64 && op == MAX) return pick_tile<i64, OpMax>(k1, in, out, outer, n1, n2, nullptr, s);
  return -1;
}

}  // namespace exsum
