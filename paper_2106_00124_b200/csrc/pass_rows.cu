// pass_rows.cu -- windowed pass along the contiguous (last) axis.
//
// Restates windowed_sum_axis (reference pkg/src/exsum/scan.py:61-102) when
// the lines are contiguous rows ([rows, n], inner == 1).
//
// B200 mapping: a warp owns a row (or, for n <= 32, floor(32/n) whole rows)
// and walks it in warp-wide steps of one element per lane, so every load and
// store is a contiguous 32-element run.  The in-block scans are done with
// warp shuffles, but NOT as log-step (Kogge-Stone) scans: the reference's
// suffix S[x] = a[x] (+) S[x+1] is right nested and its prefix
// P[x] = P[x-1] (+) a[x] is left nested, so the shuffles iterate
// "S = a (+) shfl_down(S, 1)" k-1 times, which after iteration m holds
// exactly the right-nested fold of a[x..x+m].  That keeps float results
// bit-identical to the reference at ~3 instructions per element, far below
// the instruction budget of an HBM-bound pass (B200: ~44 lane-instructions per
// f32 element at 6.5 TB/s).
//
//   k <= 32 : steps of L = k*floor(32/k) lanes hold whole blocks; the stitch
//             partner P[min(x+k-1, n-1)] lives in this step or the next one
//             (one-step look-ahead).  A prefetch ring keeps PF steps of loads
//             in flight per lane.
//   k <= 32*RMAX : a block spans ceil(k/32) steps; suffixes carry across steps
//             right to left, prefixes left to right (exactly nested), and the
//             suffixes of the current block stay in registers while the next
//             block's prefix streams by.  k == n is the whole-row suffix scan
//             (scan.py:66-68).
//   larger k : falls back to the per-block kernel in pass_strided.cu.
#include "exsum_common.cuh"
#include "exsum_launch.h"
#include "generic_blocks.cuh"

namespace exsum {


template <class T>
__device__ __forceinline__ T epi_apply(bool epi, T tot, T v) {
  return epi ? OpAdd::inverse<T>(tot, v) : v;
}

// ---------------------------------------------------------------- k <= 32 --
template <class T, class Op, int PF>
__global__ void __launch_bounds__(256)
k_rows_small(const T* __restrict__ in, T* __restrict__ out, int64_t rows, int64_t n, int k,
             int64_t seg_steps, const typename AccOf<T>::type* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const T ident = Op::template identity<T>();
  const int64_t last_bs = (int64_t)k * ((n - 1) / k);

  if (n <= 32) {
    // packed: R whole rows per warp step, every block inside one step
    const int R = 32 / (int)n;
    const int row_in = lane / (int)n;
    const int x = lane % (int)n;
    const bool is_start = x % k == 0;
    const bool is_end = (x % k == k - 1) || (x == n - 1);
    const int y = (int)(x + k - 1 < n - 1 ? x + k - 1 : n - 1);
    const int src = lane - x + y;
    const bool last = x >= last_bs;
    const int64_t groups = (rows + R - 1) / R;
    for (int64_t g = warp; g < groups; g += nwarps) {
      const int64_t row = g * R + row_in;
      const bool valid = row_in < R && row < rows;
      const T a = valid ? ld1(in + row * n + x) : ident;
      T S = a, P = a;
      for (int it = 1; it < k; ++it) {
        const T tS = shfl_down1(S);
        const T tP = shfl_up1(P);
        if (!is_end) S = Op::apply(a, tS);
        if (!is_start) P = Op::apply(tP, a);
      }
      const T Py = shfl_idx(P, src < 32 ? src : 31);
      const T o = (is_start || last) ? S : Op::apply(S, Py);
      if (valid) st1(out + row * n + x, epi_apply(epi, tot, o));
    }
    return;
  }

  const int m = 32 / k;
  const int L = m * k;
  const int64_t nsteps = (n + L - 1) / L;
  const int64_t nseg = (nsteps + seg_steps - 1) / seg_steps;
  const int64_t items = rows * nseg;
  const bool lane_ok = lane < L;
  const bool is_start = lane % k == 0;
  const bool is_end_blk = lane % k == k - 1;

  for (int64_t w = warp; w < items; w += nwarps) {
    const int64_t row = w / nseg;
    const int64_t seg = w % nseg;
    const int64_t s0 = seg * seg_steps;
    const int64_t s1 = s0 + seg_steps < nsteps ? s0 + seg_steps : nsteps;
    const int64_t s_lim = s1 < nsteps ? s1 : nsteps - 1;  // last step loaded (halo)
    const T* prow = in + row * n;
    T* orow = out + row * n;

    T ring[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int64_t s = s0 + i;
      const int64_t x = s * L + lane;
      ring[i] = (s <= s_lim && lane_ok && x < n) ? ld1(prow + x) : ident;
    }

    // scan of one step: exact nested in-block suffix / prefix
    auto scan = [&](T a, int64_t s, T& S, T& P) {
      const int64_t x = s * L + lane;
      const bool is_end = is_end_blk || x == n - 1;
      S = a;
      P = a;
      for (int it = 1; it < k; ++it) {
        const T tS = shfl_down1(S);
        const T tP = shfl_up1(P);
        if (!is_end) S = Op::apply(a, tS);
        if (!is_start) P = Op::apply(tP, a);
      }
    };

    T curS, curP;
    scan(ring[0], s0, curS, curP);
    for (int64_t s = s0; s < s1; ++s) {
      const T a_next = ring[1 % PF];
#pragma unroll
      for (int i = 0; i + 1 < PF; ++i) ring[i] = ring[i + 1];
      {
        const int64_t sp = s + PF;
        const int64_t xp = sp * L + lane;
        ring[PF - 1] = (sp <= s_lim && lane_ok && xp < n) ? ld1(prow + xp) : ident;
      }
      T nxtS = ident, nxtP = ident;
      if (s + 1 < nsteps) scan(a_next, s + 1, nxtS, nxtP);

      const int64_t x0 = s * L;
      const int64_t x = x0 + lane;
      const int64_t y = x + k - 1 < n - 1 ? x + k - 1 : n - 1;
      const int64_t rel = y - x0;
      const int src_same = rel < 32 ? (int)rel : 31;
      const int src_next = (rel - L) >= 0 && (rel - L) < 32 ? (int)(rel - L) : 0;
      const T Ps = shfl_idx(curP, src_same);
      const T Pn = shfl_idx(nxtP, src_next);
      const T Py = rel < L ? Ps : Pn;
      const bool last = x >= last_bs;
      const T o = (is_start || last) ? curS : Op::apply(curS, Py);
      if (lane_ok && x < n) st1(orow + x, epi_apply(epi, tot, o));
      curS = nxtS;
      curP = nxtP;
    }
  }
}

// ------------------------------------------------------- 32 < k <= 32*RMAX --
template <class T, class Op, int RMAX>
__global__ void __launch_bounds__(256)
k_rows_big(const T* __restrict__ in, T* __restrict__ out, int64_t rows, int64_t n, int64_t k,
           int64_t seg_blocks, const typename AccOf<T>::type* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const T ident = Op::template identity<T>();
  const int64_t nb = (n + k - 1) / k;
  const int64_t last_bs = k * ((n - 1) / k);
  const int nsb = (int)((k + 31) / 32);
  const int64_t nseg = (nb + seg_blocks - 1) / seg_blocks;
  const int64_t items = rows * nseg;

  for (int64_t w = warp; w < items; w += nwarps) {
    const int64_t row = w / nseg;
    const int64_t seg = w % nseg;
    const int64_t b0 = seg * seg_blocks;
    const int64_t b1 = b0 + seg_blocks < nb ? b0 + seg_blocks : nb;
    const T* prow = in + row * n;
    T* orow = out + row * n;

    // right-to-left suffix over the steps of one block, exactly nested
    auto block_suffix = [&](T (&v)[RMAX], int blen) {
      T carry = ident;
#pragma unroll
      for (int j = RMAX - 1; j >= 0; --j) {
        if (j < nsb) {
          const int sl = blen - 32 * j;  // valid lanes in step j
          if (sl > 0) {
            const T a = v[j];
            T S = a;
            if (lane == 31 && sl > 32) S = Op::apply(a, carry);
            for (int it = 1; it < 32; ++it) {
              const T t = shfl_down1(S);
              if (lane < 31 && lane < sl - 1) S = Op::apply(a, t);
            }
            carry = shfl_idx(S, 0);
            v[j] = S;
          }
        }
      }
    };

    T cur[RMAX];
    {
      const int64_t bs = b0 * k;
      const int blen = (int)(n - bs < k ? n - bs : k);
#pragma unroll
      for (int j = 0; j < RMAX; ++j) {
        const int r = 32 * j + lane;
        cur[j] = (j < nsb && r < blen) ? ld1(prow + bs + r) : ident;
      }
      block_suffix(cur, blen);
    }

    for (int64_t b = b0; b < b1; ++b) {
      const int64_t bs = b * k;
      if (bs == last_bs) {
        const int blen = (int)(n - bs);
#pragma unroll
        for (int j = 0; j < RMAX; ++j) {
          const int r = 32 * j + lane;
          if (j < nsb && r < blen) st1(orow + bs + r, epi_apply(epi, tot, cur[j]));
        }
        break;
      }
      const int64_t ns = bs + k;
      const bool more = b + 1 < b1;
      const int64_t avail = n - ns;
      const int64_t want = more ? k : k - 1;
      const int nlen = (int)(avail < want ? avail : want);
      T nxt[RMAX];
#pragma unroll
      for (int j = 0; j < RMAX; ++j) {
        const int r = 32 * j + lane;
        nxt[j] = (j < nsb && r < nlen) ? ld1(prow + ns + r) : ident;
      }
      // left-to-right prefix of the next block, stitched onto S of this one
      T Pcarry = ident, Pfin = ident;
#pragma unroll
      for (int j = 0; j < RMAX; ++j) {
        if (j < nsb) {
          const T a = nxt[j];
          T P = a;
          if (lane == 0 && j > 0) P = Op::apply(Pcarry, a);
          for (int it = 1; it < 32; ++it) {
            const T t = shfl_up1(P);
            if (lane > 0) P = Op::apply(t, a);
          }
          const int fin = nlen - 1 - 32 * j;
          if (fin >= 0 && fin < 32) Pfin = shfl_idx(P, fin);
          const T up = shfl_up1(P);
          const int r = 32 * j + lane;  // position in block b (a full block)
          if (r < k) {
            T o = cur[j];
            if (r > 0) {
              const T Pv = (r - 1 < nlen) ? (lane > 0 ? up : Pcarry) : Pfin;
              o = Op::apply(o, Pv);
            }
            st1(orow + bs + r, epi_apply(epi, tot, o));
          }
          Pcarry = shfl_idx(P, 31);
        }
      }
      if (!more) break;
      block_suffix(nxt, nlen);
#pragma unroll
      for (int j = 0; j < RMAX; ++j) cur[j] = nxt[j];
    }
  }
}

// ------------------------------------------- k | C, C | n: lane-owned chunks --
// The common case (every BASELINE row pass): n is a multiple of a chunk of C
// elements and C a multiple of K, so blocks never straddle chunks.  A warp
// stages 32 chunks (+1 halo chunk) of the flattened rows through shared memory
// with coalesced 16-byte loads, each lane then owns one chunk in registers and
// runs the exact in-block suffix / prefix sequentially (no shuffles), takes the
// next block's raw values for its last block from its neighbour's chunk in
// shared memory, and the results leave through shared memory again as
// coalesced 16-byte stores.  ~0.2 warp instructions per element.
// CMAX: register capacity; c_rt: the chunk when RT (runtime chunk, e.g. a
// whole 28-element row), else C == CMAX at compile time.
template <class T, class Op, int K, int CMAX, int WARPS, bool RT>
__global__ void __launch_bounds__(WARPS * 32)
k_rows_tile(const T* __restrict__ in, T* __restrict__ out, int64_t rows, int64_t n,
            const typename AccOf<T>::type* __restrict__ total, int c_rt) {
  constexpr int VE = 16 / sizeof(T);  // elements per 16-byte vector
  constexpr int CVMAX = CMAX / VE;
  constexpr int MMAX = CMAX / K;
  const int C = RT ? c_rt : CMAX;
  const int CV = C / VE;              // vectors per chunk
  // padded chunk stride, an odd number of 16-byte vectors: 16-byte accesses of
  // 8 consecutive lanes land in 8 distinct bank groups
  const int STRIDE = ((CV + 1) | 1) * VE;
  // v / CV by multiply-shift: exact for v < 65536 / CV (v <= 33 * CV here)
  const unsigned cv_magic = (65536u + (unsigned)CV - 1) / (unsigned)CV;
  const int M = C / K;                // blocks per chunk
  static_assert(CMAX % K == 0 && CMAX % VE == 0, "chunk shape");
  static_assert(CVMAX <= 32, "the multiply-shift division below is exact for CV <= 32");
  typedef Vec<T, VE> VT;
  // wide chunks (CVMAX > 8, e.g. f64 k = 32) would hold two chunks of
  // registers at once to prefetch: they double-buffer the stage instead, the
  // next tile's 16-byte cp.async copies in flight while this one is computed
  constexpr bool PREFETCH = CVMAX <= 8;
  constexpr int SLOT = 33 * (CMAX + 2 * VE);  // one staged tile, padded chunks
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  T* smw = reinterpret_cast<T*>(smem_raw) + wib * (PREFETCH ? 1 : 2) * SLOT;
  T* sm = smw;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t cpr = n / C;  // chunks per row
  const int64_t nchunks = rows * cpr;
  const int64_t ntiles = (nchunks + 31) / 32;

  // each lane's share of a tile's 16-byte vectors, held in registers so the
  // next tile's loads are in flight while this one is computed (PREFETCH)
  constexpr int PV = (33 * CVMAX + 31) / 32;
  VT pre[PREFETCH ? PV : 1];
  auto load_tile = [&](int64_t t) {
    if constexpr (!PREFETCH) return;
    if (t >= ntiles) return;
    const int64_t a0 = nchunks - t * 32;
    const int nl = a0 >= 33 ? 33 : (int)a0;
    const VT* src = reinterpret_cast<const VT*>(in + t * 32 * C);
#pragma unroll
    for (int i = 0; i < PV; ++i) {
      const int v = lane + 32 * i;
      if (v < nl * CV) pre[i] = ld_stream<T, VE>(reinterpret_cast<const T*>(src + v));
    }
  };
  // !PREFETCH: the tile's vectors straight into stage slot `slot` by cp.async
  auto copy_tile = [&](int64_t t, int slot) {
    if (t < ntiles) {
      const int64_t a0 = nchunks - t * 32;
      const int nl = a0 >= 33 ? 33 : (int)a0;
      const VT* src = reinterpret_cast<const VT*>(in + t * 32 * C);
      T* dstm = smw + slot * SLOT;
      for (int v = lane; v < nl * CV; v += 32) {
        const int cq = (int)(((unsigned)v * cv_magic) >> 16);  // v / CV
        cp_async16(dstm + cq * STRIDE + (v - cq * CV) * VE, src + v);
      }
    }
    cp_async_commit();
  };
  if (PREFETCH) load_tile(warp);
  else copy_tile(warp, 0);
  int slot = 0;

  for (int64_t tile = warp; tile < ntiles; tile += nwarps) {
    const int64_t c0 = tile * 32;
    const int64_t avail = nchunks - c0;  // chunks left from c0 (>= 1)
    const int nload = avail >= 33 ? 33 : (int)avail;
    if constexpr (PREFETCH) {
#pragma unroll
      for (int i = 0; i < PV; ++i) {
        const int v = lane + 32 * i;
        if (v < nload * CV) {
          const int cq = (int)(((unsigned)v * cv_magic) >> 16);  // v / CV (v < 4096)
          *reinterpret_cast<VT*>(sm + cq * STRIDE + (v - cq * CV) * VE) = pre[i];
        }
      }
      __syncwarp();
      load_tile(tile + nwarps);
    } else {
      sm = smw + slot * SLOT;
      copy_tile(tile + nwarps, slot ^ 1);  // the slot the previous tile left
      cp_async_wait<1>();                  // this tile's copies have landed
      __syncwarp();
    }
    const int64_t c = c0 + lane;
    const bool valid = lane < nload && lane < 32 && c < nchunks;
    const int64_t xc = valid ? (c % cpr) * C : 0;  // chunk start within its row
    T a[CMAX];
#pragma unroll
    for (int v = 0; v < CVMAX; ++v) {
      if (v < CV) {
        const VT q = *reinterpret_cast<const VT*>(sm + lane * STRIDE + v * VE);
#pragma unroll
        for (int j = 0; j < VE; ++j) a[v * VE + j] = q.v[j];
      }
    }
    const bool has_next_chunk = valid && xc + C < n;  // next block in the same row
    const T* nbp = sm + (lane + 1) * STRIDE;          // neighbour's raw chunk (read-only)
    // blocks in ascending order: S in place (right nested), then the stitch
    // with the next block's left-nested prefix (raw, not yet overwritten)
#pragma unroll
    for (int j = 0; j < MMAX; ++j) {
      if (j >= M) break;
#pragma unroll
      for (int r = K - 2; r >= 0; --r) a[j * K + r] = Op::apply(a[j * K + r], a[j * K + r + 1]);
      const int64_t xs = xc + j * K;
      const bool last = xs + K >= n;  // n % K == 0: the last block is full
      if (!last) {
        const bool inner = j + 1 < M;
        T P = inner ? a[(j + 1) * K] : (has_next_chunk ? nbp[0] : a[0]);
#pragma unroll
        for (int r = 1; r < K; ++r) {
          if (r >= 2) P = Op::apply(P, inner ? a[(j + 1) * K + r - 1] : nbp[r - 1]);
          a[j * K + r] = Op::apply(a[j * K + r], P);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < CVMAX; ++v) {
      if (v < CV) {
        VT q;
#pragma unroll
        for (int jj = 0; jj < VE; ++jj) {
          const T w = a[v * VE + jj];
          q.v[jj] = epi ? OpAdd::inverse<T>(tot, w) : w;
        }
        *reinterpret_cast<VT*>(sm + lane * STRIDE + v * VE) = q;
      }
    }
    __syncwarp();
    const int nstore = avail >= 32 ? 32 : (int)avail;
    VT* dst = reinterpret_cast<VT*>(out + c0 * C);
#pragma unroll 4
    for (int v = lane; v < nstore * CV; v += 32)
      st_stream<T, VE>(reinterpret_cast<T*>(dst + v),
                       *reinterpret_cast<const VT*>(sm + (((unsigned)v * cv_magic) >> 16) * STRIDE +
                                                    (v - (int)(((unsigned)v * cv_magic) >> 16) * CV) * VE));
    __syncwarp();
    slot ^= 1;
  }
  if constexpr (!PREFETCH) cp_async_wait<0>();
}

// ---------------------------------------------- k == n > 32: whole-row suffix --
// scan.py:66-68 (k >= n is a reverse inclusive scan).  The exact right-nested
// suffix is one dependent chain per row, so the parallelism is across rows:
// lane = row.  A warp walks its 32 rows right to left in chunks of W elements
// staged (coalesced) through padded shared memory; each lane runs its row's
// chain through the chunk and the chunk leaves coalesced.
template <class T, class Op, int W, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
k_rows_suffix(const T* __restrict__ in, T* __restrict__ out, int64_t rows, int64_t n,
              const typename AccOf<T>::type* __restrict__ total) {
  static_assert(W == 32, "one chunk column per lane");
  constexpr int STRIDE = W + 1;
  __shared__ T smem[WARPS][32 * STRIDE];
  const int lane = threadIdx.x & 31;
  T* sm = smem[threadIdx.x >> 5];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t groups = (rows + 31) / 32;
  for (int64_t g = warp; g < groups; g += nwarps) {
    const int64_t r0 = g * 32;
    const int nr = rows - r0 >= 32 ? 32 : (int)(rows - r0);
    // chunks of W columns from the row end; 32 independent loads per chunk,
    // the next chunk's loads issued while the current one is scanned
    T v[32];
    {
      const int64_t xs = n - W > 0 ? n - W : 0;
      const int64_t x = xs + lane;
      if (nr == 32 && x < n) {  // unpredicated: all 32 loads in flight at once
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = ld1(in + (r0 + r) * n + x);
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = (r < nr && x < n) ? ld1(in + (r0 + r) * n + x) : T(0);
      }
    }
    T S = T(0);
    for (int64_t xe = n; xe > 0; xe -= W) {
      const int64_t xs = xe - W > 0 ? xe - W : 0;
      const int w = (int)(xe - xs);
#pragma unroll
      for (int r = 0; r < 32; ++r) sm[r * STRIDE + lane] = v[r];
      __syncwarp();
      if (xs > 0) {
        const int64_t ns = xs - W > 0 ? xs - W : 0;
        const int64_t x = ns + lane;
        if (nr == 32 && x < xs) {
#pragma unroll
          for (int r = 0; r < 32; ++r) v[r] = ld1(in + (r0 + r) * n + x);
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) v[r] = (r < nr && x < xs) ? ld1(in + (r0 + r) * n + x) : T(0);
        }
      }
      if (lane < nr) {
        int x = w - 1;
        if (xe == n) {
          S = sm[lane * STRIDE + x];
          --x;
        }
        for (; x >= 0; --x) {
          S = Op::apply(sm[lane * STRIDE + x], S);
          sm[lane * STRIDE + x] = S;
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r < nr && lane < w) {
          const T t = sm[r * STRIDE + lane];
          st1(out + (r0 + r) * n + xs + lane, epi ? OpAdd::inverse<T>(tot, t) : t);
        }
      __syncwarp();
    }
  }
}

namespace {

template <class T, class Op, int K, int C, bool RT = false>
int go_tile(const T* in, T* out, int64_t rows, int64_t n, const typename AccOf<T>::type* total,
            cudaStream_t s, int c_rt = C) {
  constexpr int WARPS = 4;
  const int64_t tiles = (rows * (n / c_rt) + 31) / 32;
  int64_t grid = (tiles + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  constexpr int VE = 16 / (int)sizeof(T);
  constexpr bool PREFETCH = C / VE <= 8;
  const size_t smem = (size_t)WARPS * (PREFETCH ? 1 : 2) * 33 * (C + 2 * VE) * sizeof(T);
  ensure_smem((const void*)k_rows_tile<T, Op, K, C, WARPS, RT>, smem);
  k_rows_tile<T, Op, K, C, WARPS, RT><<<(unsigned)grid, WARPS * 32, smem, s>>>(in, out, rows, n,
                                                                              total, c_rt);
  return 1;
}

// chunk C (elements per lane): a multiple of K and of the 16-byte vector,
// >= 32 bytes, preferring 64-128 bytes; it must divide n
constexpr int chunk_base(int K, int VE, int es) {
  int c = K > VE ? K : VE;  // lcm of powers of two
  while (c * es < 32) c *= 2;
  return c;
}

template <class T, class Op, int K>
int try_tile(const T* in, T* out, int64_t rows, int64_t n, const typename AccOf<T>::type* total,
             cudaStream_t s) {
  constexpr int VE = 16 / sizeof(T);
  constexpr int C0 = chunk_base(K, VE, (int)sizeof(T));
  constexpr int C2 = 2 * C0;
  const uintptr_t al = (uintptr_t)in | (uintptr_t)out;
  if (al % 16) return -1;
  if constexpr (C2 * sizeof(T) <= 128) {
    if (n % C2 == 0) return go_tile<T, Op, K, C2>(in, out, rows, n, total, s);
  }
  if constexpr (C0 * sizeof(T) <= 256) {
    if (n % C0 == 0) return go_tile<T, Op, K, C0>(in, out, rows, n, total, s);
  }
  // one (short) row per chunk: n a multiple of K and of the vector, <= 32 elements
  if constexpr (32 % K == 0 && 32 % VE == 0) {
    if (n <= 32 && n % K == 0 && n % VE == 0 && (size_t)n * sizeof(T) >= 32)
      return go_tile<T, Op, K, 32, true>(in, out, rows, n, total, s, (int)n);
  }
  return -1;
}

template <class T, class Op>
int go_rows(const T* in, T* out, int64_t rows, int64_t n, int64_t k,
            const typename AccOf<T>::type* total, cudaStream_t s) {
  const int64_t want_warps = (int64_t)num_sms() * 64;
  {
    int rc = -1;
    switch (k) {
      case 2: rc = try_tile<T, Op, 2>(in, out, rows, n, total, s); break;
      case 4: rc = try_tile<T, Op, 4>(in, out, rows, n, total, s); break;
      case 8: rc = try_tile<T, Op, 8>(in, out, rows, n, total, s); break;
      case 16: rc = try_tile<T, Op, 16>(in, out, rows, n, total, s); break;
      case 32: rc = try_tile<T, Op, 32>(in, out, rows, n, total, s); break;
      default: break;
    }
    if (rc >= 0) return rc;
  }
  if (k == n && k > 32) {
    constexpr int WARPS = 4;
    const int64_t groups = (rows + 31) / 32;
    int64_t grid = (groups + WARPS - 1) / WARPS;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    k_rows_suffix<T, Op, 32, WARPS><<<(unsigned)grid, WARPS * 32, 0, s>>>(in, out, rows, n, total);
    return 1;
  }
  if (k <= 32) {
    int64_t seg_steps = 1;
    int64_t items;
    if (n <= 32) {
      items = (rows + (32 / n) - 1) / (32 / n);
    } else {
      const int64_t L = k * (32 / k);
      const int64_t nsteps = (n + L - 1) / L;
      int64_t nseg = (want_warps + rows - 1) / rows;
      int64_t max_seg = nsteps / 8;
      if (max_seg < 1) max_seg = 1;
      if (nseg > max_seg) nseg = max_seg;
      seg_steps = (nsteps + nseg - 1) / nseg;
      items = rows * ((nsteps + seg_steps - 1) / seg_steps);
    }
    int64_t grid = (items * 32 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 32;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    k_rows_small<T, Op, 4><<<(unsigned)grid, 256, 0, s>>>(in, out, rows, n, (int)k, seg_steps,
                                                         total);
    return 1;
  }
  const int nsb = (int)((k + 31) / 32);
  const int64_t nb = (n + k - 1) / k;
  int64_t nseg = (want_warps + rows - 1) / rows;
  int64_t max_seg = nb / 4;
  if (max_seg < 1) max_seg = 1;
  if (nseg > max_seg) nseg = max_seg;
  const int64_t seg_blocks = (nb + nseg - 1) / nseg;
  const int64_t items = rows * ((nb + seg_blocks - 1) / seg_blocks);
  int64_t grid = (items * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
#define EXSUM_ROWS_BIG(R)                                                              \
  if (nsb <= R) {                                                                      \
    k_rows_big<T, Op, R><<<(unsigned)grid, 256, 0, s>>>(in, out, rows, n, k, seg_blocks, \
                                                        total);                        \
    return 1;                                                                          \
  }
  EXSUM_ROWS_BIG(2)
  EXSUM_ROWS_BIG(4)
  EXSUM_ROWS_BIG(8)
  EXSUM_ROWS_BIG(16)
  if (sizeof(T) == 4) { EXSUM_ROWS_BIG(32) }
#undef EXSUM_ROWS_BIG
  // very large k: per-block sweeps (one thread per (row, block))
  const int64_t items2 = rows * nb;
  int64_t grid2 = (items2 + 255) / 256;
  const int64_t cap2 = (int64_t)num_sms() * 64;
  if (grid2 > cap2) grid2 = cap2;
  k_strided_blocks<T, Op, 1><<<(unsigned)grid2, 256, 0, s>>>(in, out, rows, n, 1, k, total);
  return 1;
}

}  // namespace

int launch_rows_pass(int dtype, int op, const void* in, void* out, int64_t rows, int64_t n,
                     int64_t k, const void* total, cudaStream_t s) {
  if (dtype == F32 && op == ADD)
    return go_rows<float, OpAdd>((const float*)in, (float*)out, rows, n, k, (const double*)total, s);
  if (dtype == F64 && op == ADD)
    return go_rows<double, OpAdd>((const double*)in, (double*)out, rows, n, k,
                                  (const double*)total, s);
  if (dtype == I64 && op == ADD)
    return go_rows<i64, OpAdd>((const i64*)in, (i64*)out, rows, n, k, (const i64*)total, s);
  if (dtype == I64 && op == MAX)
    return go_rows<i64, OpMax>((const i64*)in, (i64*)out, rows, n, k, nullptr, s);
  return -2;
}

}  // namespace exsum
