// fused_pair.cuh -- the last two axes in one pass over HBM.
//
// Fuses the windowed pass along axis d-2 (scan.py:61-102, strided) with the
// row operation along the contiguous axis d-1:
//   ROW_WIN  : the windowed pass along axis d-1 (bdbs_included's last two
//              passes, included.py:127-128; with the BDBSC complement epilogue,
//              excluded.py:72-75)
//   ROW_EXCL : the box-complement round of the peeled last axis,
//              out = P[x-1] (+) S[x+k] (+) T[row] (excluded.py:151-156 restated;
//              see exsum_capi.cu)
// so the intermediate array never goes back to HBM: 2*N*s bytes instead of 4.
//
// B200 mapping: one CTA owns a slab [x1-segment, full rows] of one outer index
// and streams it in blocks of k1 rows:
//   * every thread owns one 16-byte column vector of the row and prefetches
//     its own vectors of blocks b+2, b+3 with cp.async (LDGSTS) into a 2-slot
//     shared ring -- no CTA barrier is needed for the loads, and two blocks of
//     loads (128 KB at the C4 shape) are in flight while block b is processed;
//   * the axis-(d-2) pass runs in registers exactly as in pass_strided.cu
//     (suffix of block b, running prefix of block b+1), writing the k1 output
//     rows to a shared stage laid out conflict-free for both access patterns
//     (chunk stride an odd number of 16-byte vectors, or an XOR swizzle of
//     the vectors where chunks are narrower than 8 vectors -- fp_swz);
//   * after one __syncthreads each warp takes whole rows, each lane a chunk of
//     C = n2/32 consecutive elements in registers, and runs the row op
//     (sequential exact in-block scans for ROW_WIN; lane fold + warp scans for
//     ROW_EXCL), writing back in place; after a second __syncthreads the rows
//     leave as coalesced 16-byte stores.
// Float association: ROW_WIN keeps the reference's nesting, so BDBS stays
// bit-exact; ROW_EXCL is reassociated (tolerance).
#pragma once

#include <stdlib.h>

#include <type_traits>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

// K1: window along axis d-2 (compile time); the ROW_WIN row op uses the same
// window along the row (K2 == K1, the cubic boxes of the BASELINE configs);
// ROW_EXCL takes any shift kx at run time.
#ifndef FP_EXCL_BLK
#define FP_EXCL_BLK 1
#endif
#ifndef FP_NARROW_C
#define FP_NARROW_C 8
#endif
// largest window along the row that takes 256-column strips on long rows
#ifndef FP_STRIP_NARROW_K8
#define FP_STRIP_NARROW_K8 8
#endif
#ifndef FP_STRIP_NARROW_K4
#define FP_STRIP_NARROW_K4 2
#endif
// the stores of unit u's rows run inside unit u+1's axis-(d-2) pass, each row
// right before its stage slot is rewritten (interleaving the streaming stores
// with the compute instead of a store-only loop after the row op).  Measured
// per mode and shape: the box-complement row rounds gain everywhere (C4 f32
// BLK 1.414 -> 1.322 ms, C5 f64 -30 us, C4 4^3 -45 us), ROW_WIN gains on
// 8-byte rows (C5 f64 box 8^3 / 16^3 -25 us), narrow float32 rows and k = 4
// (C4 box 4^3 -36 us) but loses on 1024-wide float32 rows with k >= 8 (C4 BDBS
// 1.335 -> 1.408 ms): those keep the store loop after the row op (WIN_SLOW)
#ifndef FP_DEFER_STORE
#define FP_DEFER_STORE 1  // 1: every mode but WIN_SLOW below; 2: every mode
#endif
// balanced unit ranges instead of uniform segments (go_pair): threshold in
// percent over the even split, ranges per SM; EXSUM_FP_BALANCED=0 turns it off
#ifndef FP_BALANCED_PCT
#define FP_BALANCED_PCT 2
#endif
// windows along axis d-2 below this keep uniform segments under ROW_WIN
// (measured: C5 f64 box 4^3 0.355 -> 0.364 ms, 2^3 0.353 -> 0.374 ms in balanced
// mode; box 8^3 0.361 -> 0.340, 16^3 0.381 -> 0.363; the row rounds of
// box-complement gain at every window: C5 box 2^3 0.384 -> 0.365)
#ifndef FP_BALANCED_MIN_K_WIN
#define FP_BALANCED_MIN_K_WIN 8
#endif
#ifndef FP_BALANCED_MULT
#define FP_BALANCED_MULT 1
#endif
#ifndef FP_BALANCED_TAIL
#define FP_BALANCED_TAIL 1
#endif
// strips (rows longer than the widest row template) take the balanced schedules too
#ifndef FP_BALANCED_STRIPS
#define FP_BALANCED_STRIPS 1
#endif
// EXSUM_FP_BALANCED: 0 off, 1 (default) by the cost model, 2 whenever the
// kernel allows it (tests: balanced ranges on small arrays, every window)
inline int fp_balanced_mode() {
  const char* e = getenv("EXSUM_FP_BALANCED");
  return e && e[0] >= '0' && e[0] <= '2' ? e[0] - '0' : 1;
}
// Rows per streaming unit: 16 (a multiple of K1) for wide rows; narrow rows
// (C <= 8: 64-thread CTAs whose shared ring and stage bound the CTAs per SM)
// take 8-row units where K1 allows, doubling the resident CTAs.
__host__ __device__ constexpr int fp_unit_rows(int C, int K1) {
  return (C <= FP_NARROW_C && K1 <= 4) ? 4 : (C <= FP_NARROW_C && K1 <= 8) ? 8
                                                : (16 / K1 > 0 ? 16 / K1 : 1) * K1;
}

// Stage layout: a row of 16-byte vectors with vector v stored at
// v ^ ((v >> 3) & (CV - 1)) (CV = vectors per lane chunk).  Within every
// aligned group of 8 vectors this is a permutation, so the streaming phase
// (thread t <-> vector t) stays conflict-free, and the row op's stride-CV
// accesses (lane L <-> vector CV*L + c, any shift c) hit 8 distinct 16-byte
// bank groups per quarter warp -- padding the chunks (the previous layout)
// left a 2-way conflict on the streaming side whenever CV < 8.
template <int CV>
__device__ __forceinline__ int fp_swz(int v) {
  return v ^ ((v >> 3) & (CV - 1));
}
// (strips keep the padded layout: their halo lives in a 33rd chunk)
__host__ __device__ constexpr bool fp_swizzled(int CV, int MODE, bool STRIP = false) {
  return CV < 8 && MODE != ROW_EXCL && !STRIP;
}
// chunk stride in 16-byte vectors: CV when swizzled, else padded to odd
__host__ __device__ constexpr int fp_chunk_stride(int CV, int MODE, bool STRIP = false) {
  return fp_swizzled(CV, MODE, STRIP) ? CV : ((CV + 1) | 1);
}

template <class T, class Op, int C, int K1, int MODE, int TV, bool STRIP>
// narrow rows ask for more resident CTAs: a register cap that raises the warps
// per SM there (4-byte, 64-thread CTAs: 12, C3b 0.033 -> 0.030 ms; 8-byte,
// 128 threads: 4, C2 0.066 -> 0.062 ms, except the max row op, which spills)
// STRIP (ROW_WIN on rows longer than 32 C): the CTA takes a strip of 32 C
// columns plus a right halo of K1 - 1 columns streamed by one extra warp, so
// the row op's last block sees its neighbour block; the halo's outputs belong
// to the next strip and are not stored
__global__ void __launch_bounds__(32 * C / TV + (STRIP ? 32 : 0),
                                   (C <= 8 ? (sizeof(T) == 4 ? (MODE == ROW_EXCL_BLK && K1 >= 8 ? 8 : 12)
                                                  : (MODE == ROW_EXCL ? 1 : 4)) : 1))
k_fused_pair(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n1,
             int64_t kx, int64_t seg_len, int64_t nseg,
             const typename AccOf<T>::type* __restrict__ total, const T* __restrict__ Tail,
             int64_t n2full, int64_t nstrips, int64_t bal_line0, int bal_ctas) {
  constexpr int VE = 16 / sizeof(T);  // 16-byte vector (stage layout, row op)
  constexpr int N2 = 32 * C;           // row length
  constexpr int NT = N2 / TV;          // threads: one TV-element column vector each
  constexpr int NW = NT / 32;
  constexpr int CV = C / VE;           // vectors per lane chunk
  // stage layout (fp_stage): XOR-swizzled rows where chunks are narrower
  // than 8 vectors (the padded layout conflicts 2-way there on the streaming
  // side) except under the prefix/suffix row op, whose many chunk accesses
  // would each pay the lane-dependent swizzle in address arithmetic (C2 max
  // 0.084 -> 0.090 ms); padded chunks (odd stride) otherwise
  constexpr bool SWZ = fp_swizzled(CV, MODE, STRIP);
  constexpr int CH = fp_chunk_stride(CV, MODE, STRIP) * VE;  // chunk stride (elements)
  constexpr int HV = STRIP ? (K1 - 1 + VE - 1) / VE : 0;  // halo vectors per row
  constexpr int RAWP = N2 + HV * VE;                 // ring row pitch
  constexpr int ROWP = (STRIP ? 33 : 32) * CH;       // stage row length (elements; chunk 32 = halo)
  // stage offset of element e of a row / of vector v of lane L's chunk
  auto eoff = [](int64_t e) -> int64_t {
    if constexpr (SWZ) return fp_swz<CV>((int)(e / VE)) * VE + (e % VE);
    else return (e / C) * CH + (e % C);
  };
  constexpr int K2 = K1;
  constexpr int M2 = C / K2;           // row-op blocks per lane chunk
  constexpr int G = fp_unit_rows(C, K1) / K1;  // blocks per unit
  constexpr int U = G * K1;            // rows per unit: register tile, stage, prefetch granule
  static_assert(C % VE == 0 && C % K2 == 0, "shape");
  typedef Vec<T, VE> VT;  // row-op vectors
  typedef Vec<T, TV> CT;  // column vectors of the axis-(d-2) pass
  extern __shared__ __align__(16) unsigned char smem[];
  T* raw = reinterpret_cast<T*>(smem);  // [2][U][RAWP]
  T* wst = raw + 2 * U * RAWP;          // [U][ROWP]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool halo_thr = STRIP && tid >= NT;   // the halo warp
  const int hv = tid - NT;                    // its column vector
  const bool colthr = !halo_thr || hv < HV;   // owns a column vector
  const int col = halo_thr ? N2 + hv * TV : tid * TV;
  static_assert(TV == VE, "the stage swizzle assumes 16-byte column vectors");
  static_assert(!STRIP || (!SWZ && MODE == ROW_WIN && HV * VE <= CH), "strip layout");
  const int pcol = halo_thr ? 32 * CH + hv * VE
                            : SWZ ? fp_swz<CV>(tid) * VE : (col / C) * CH + (col % C);  // this thread's column vector in a stage row
  const T ident = Op::template identity<T>();
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t last_bs = (int64_t)K1 * ((n1 - 1) / K1);
  // row stride and strip count: compile-time without strips (the stride
  // stays an immediate in the streaming loops)
  const int64_t rs = STRIP ? n2full : (int64_t)N2;
  const int64_t nst = STRIP ? nstrips : 1;
  const int64_t items = outer * nseg * nst;
  const bool kvec = (kx % VE) == 0;

  // Balanced ranges (bal_ctas > 0, no strips): the lines [0, bal_line0) run as
  // uniform (line, segment) items on the first gridDim.x - bal_ctas CTAs; the
  // units of the lines from bal_line0 on are cut into bal_ctas equal
  // contiguous ranges, one per CTA, each walked as one piece per line it
  // touches.  bal_line0 = 0: the whole array that way (few lines on one
  // resident CTA per SM -- a shard's 128 planes, C5's 512 -- otherwise lose a
  // fraction of a wave or pay a halo per short segment); bal_line0 = whole
  // waves of lines: only the last partial wave is balanced.
  const int64_t gu = (int64_t)gridDim.x - bal_ctas;
  // (with strips a line is one strip of one outer index, strips fastest)
  const bool bal = bal_ctas > 0 && (int64_t)blockIdx.x >= gu;
  const int64_t nun = (n1 + U - 1) / U;  // units per line
  const int64_t bal_units = (outer * nst - bal_line0) * nun;
  int64_t item = bal ? bal_units * ((int64_t)blockIdx.x - gu) / bal_ctas : (int64_t)blockIdx.x;
  const int64_t item_end = bal ? bal_units * ((int64_t)blockIdx.x - gu + 1) / bal_ctas
                               : (bal_ctas > 0 ? bal_line0 * nseg : items);
  while (item < item_end) {
    int64_t strip, o, xs, xe;
    if (bal) {
      const int64_t l = item / nun, us = item - l * nun;
      const int64_t cnt = nun - us < item_end - item ? nun - us : item_end - item;
      strip = STRIP ? (bal_line0 + l) % nst : 0;
      o = STRIP ? (bal_line0 + l) / nst : bal_line0 + l;
      xs = us * U;
      xe = (us + cnt) * U < n1 ? (us + cnt) * U : n1;
      item += cnt;
    } else {
      // strips fastest: the CTAs in flight cover whole rows
      strip = STRIP ? item % nst : 0;
      const int64_t os = STRIP ? item / nst : item;
      o = os / nseg;
      const int64_t seg = os % nseg;
      xs = seg * seg_len;  // multiple of U
      xe = xs + seg_len < n1 ? xs + seg_len : n1;
      item += bal_ctas > 0 ? gu : (int64_t)gridDim.x;
    }
    const bool last_strip = strip + 1 == nst;
    const bool loads = colthr && !(halo_thr && last_strip);  // no halo past the row end
    const int64_t u0 = xs / U;
    const int64_t u_end = (xe + U - 1) / U;
    const T* src = in + o * n1 * rs + strip * N2 + col;
    T* dst = out + o * n1 * rs + strip * N2 + col;

    // rows loaded for unit ui: the whole unit inside the segment; past the
    // segment only the first block's K1-1 rows (the stitch partner)
    auto rows_of = [&](int64_t ui) -> int {
      const int64_t avail = n1 - ui * U;
      const int64_t want = ui >= u_end ? K1 - 1 : U;
      return (int)(avail < want ? (avail > 0 ? avail : 0) : want);
    };
    auto issue = [&](int64_t ui) {
      const int rows = rows_of(ui);
      T* d = raw + ((ui - u0) & 1) * (U * RAWP) + col;
      if (loads)
        for (int r = 0; r < rows; ++r) cp_async_n<TV * sizeof(T)>(d + r * RAWP, src + (ui * U + r) * rs);
      cp_async_commit();  // always commit: uniform group accounting
    };

    issue(u0);
    issue(u0 + 1);
    cp_async_wait<1>();
    CT cur[U];  // raw rows of the current unit (block j's rows become S in turn)
    int len = rows_of(u0);
#pragma unroll
    for (int r = 0; r < U; ++r)
      if (r < len) cur[r] = *reinterpret_cast<const CT*>(raw + col + r * RAWP);
    issue(u0 + 2);

    constexpr bool WIN_SLOW = MODE == ROW_WIN && sizeof(T) == 4 && C == 32 && K1 >= 8;
#ifndef FP_DEFER_STRIP
#define FP_DEFER_STRIP 0
#endif
    constexpr bool DEFER = (!STRIP || FP_DEFER_STRIP) &&
                           (FP_DEFER_STORE == 2 || (FP_DEFER_STORE == 1 && !WIN_SLOW));
    int prev_rows = 0;     // rows of the previous unit still in the stage (DEFER)
    int64_t prev_us = 0;
    // write row `r` of this unit's axis-(d-2) result to the stage; DEFER first
    // stores the previous unit's row r from that slot
    auto stage_put = [&](int r, const CT& v) {
      if constexpr (DEFER) {
        if (r < prev_rows && !halo_thr)
          st_stream<T, TV>(dst + (prev_us + r) * rs, *reinterpret_cast<const CT*>(wst + r * ROWP + pcol));
      }
      if (colthr) *reinterpret_cast<CT*>(wst + r * ROWP + pcol) = v;
    };

    for (int64_t u = u0; u < u_end; ++u) {
      const int64_t us = u * U;
      const int rows_u = len;
      // prefetch this warp's row tails now: they are consumed after the
      // streaming phase and would otherwise stall the row op on a global load
      constexpr int RPW = (U + NW - 1) / NW;  // rows per warp in the row op
      T tails[RPW];
      if constexpr (MODE != ROW_WIN) {
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          const int rr = warp + i * NW;
          tails[i] = (Tail && rr < rows_u) ? Tail[o * n1 + us + rr] : ident;
        }
      }
      // the next unit's rows, all at once into registers; the stitch of the
      // last block reads them there.  ROW_WIN keeps the whole next unit in
      // registers across the row op (its slot is refilled right away);
      // ROW_EXCL's row op needs those registers, so it keeps only the stitch
      // rows and reloads the unit after the row op.
      constexpr bool EARLY = true;
      constexpr int NX = EARLY ? U : K1;
      const int nlen_u = rows_of(u + 1);
      const T* sn = raw + ((u + 1 - u0) & 1) * (U * RAWP) + col;
      CT nxt[NX];
      if (nlen_u > 0) {
        cp_async_wait<1>();  // unit u+1 has landed (u+2 may still be in flight)
#pragma unroll
        for (int r = 0; r < NX; ++r)
          if (r < nlen_u) nxt[r] = *reinterpret_cast<const CT*>(sn + r * RAWP);
      }
      if constexpr (EARLY) issue(u + 3);  // refills the slot unit u+1 just vacated
#pragma unroll
      for (int jb = 0; jb < G; ++jb) {
        const int64_t bs = us + (int64_t)jb * K1;
        if (jb * K1 < rows_u) {
          const int blen = (int)(n1 - bs < K1 ? n1 - bs : K1);
          // in-block suffix S (right nested), in place
#pragma unroll
          for (int r = K1 - 2; r >= 0; --r)
            if (r < blen - 1) {
#pragma unroll
              for (int j = 0; j < TV; ++j)
                cur[jb * K1 + r].v[j] = Op::apply(cur[jb * K1 + r].v[j], cur[jb * K1 + r + 1].v[j]);
            }
          if (bs == last_bs) {  // last block of axis d-2: W = S
#pragma unroll
            for (int r = 0; r < K1; ++r)
              if (r < blen) stage_put(jb * K1 + r, cur[jb * K1 + r]);
          } else {
            // stitch with the next block's left-nested prefix (raw)
            const int64_t nrows = n1 - bs - K1;
            const int nlen = (int)(nrows < K1 ? nrows : K1);
            stage_put(jb * K1, cur[jb * K1]);
            const int nb0 = jb + 1 < G ? (jb + 1) * K1 : 0;  // in range for the dead branch
            CT P = jb + 1 < G ? cur[nb0] : nxt[0];
#pragma unroll
            for (int r = 1; r < K1; ++r) {
              const int jj = r - 1;
              if (jj >= 1 && jj < nlen) {
                const CT av = jb + 1 < G ? cur[nb0 + jj] : nxt[jj];
#pragma unroll
                for (int j = 0; j < TV; ++j) P.v[j] = Op::apply(P.v[j], av.v[j]);
              }
              CT w;
#pragma unroll
              for (int j = 0; j < TV; ++j) w.v[j] = Op::apply(cur[jb * K1 + r].v[j], P.v[j]);
              stage_put(jb * K1 + r, w);
            }
          }
        }
      }
      if constexpr (DEFER) {
        // rows of the previous unit this (shorter) unit did not overwrite
        for (int r = rows_u; r < (halo_thr ? 0 : prev_rows); ++r)
          st_stream<T, TV>(dst + (prev_us + r) * rs, *reinterpret_cast<const CT*>(wst + r * ROWP + pcol));
      }
      len = nlen_u;
      if constexpr (EARLY) {
        if (u + 1 < u_end) {
#pragma unroll
          for (int r = 0; r < U; ++r) cur[r] = nxt[r];
        }
      }
      __syncthreads();

      // ---- row operation on the rows_u rows of the stage (warp per row) ----
      // ROW_EXCL: one row at a time (two interleaved rows exceed 255
      // registers); ROW_WIN: unrolled, rows interleave for ILP
#pragma unroll (MODE == ROW_EXCL ? 1 : RPW)
      for (int ri = 0; ri < RPW; ++ri) {
        const int rr = warp + ri * NW;
        if (rr >= rows_u || (STRIP && warp >= NW)) break;
        T* wrow = wst + rr * ROWP;
        T* mine = wrow + lane * CH;  // padded layout: this lane's chunk
        // vector v of lane L's chunk (L = lane or lane + 1)
        auto cvec = [&](int L, int v) -> T* {
          if constexpr (SWZ) return wrow + fp_swz<CV>(L * CV + v) * VE;
          else return mine + (L - lane) * CH + v * VE;
        };
        T a[C];
#pragma unroll
        for (int v = 0; v < CV; ++v) {
          const VT q = *reinterpret_cast<const VT*>(cvec(lane, v));
#pragma unroll
          for (int j = 0; j < VE; ++j) a[v * VE + j] = q.v[j];
        }
        // ROW_EXCL with + and a cubic box: along a row the excluded window sum
        // is (row total) - (window), so the exact windowed row op plus one
        // warp reduction replaces the prefix/suffix scans (the float error
        // scales with the row total, inside the box-complement bound of
        // tests/parity.py); max has no inverse and keeps the scans below.
        // 8-byte rows with K2 >= 8 spill on this path (f64 512^3 box 16^3:
        // 0.58 vs 0.53 ms), so they keep the sub-chunk scans below.
        // (go_fused selects ROW_EXCL_ADD for + with kx == K2 and either 4-byte
        // elements or K2 <= 4; it runs unrolled over the warp's rows like ROW_WIN)
        constexpr bool ADD_EXCL = MODE == ROW_EXCL_ADD;
        if constexpr (MODE == ROW_WIN || ADD_EXCL) {
          T rtot = T(0);
          // exact in-block scans along the row (blocks of K2 inside the chunk)
          constexpr int NBV = (K2 + VE - 1) / VE;
          VT nbv[NBV];  // neighbour's first block, raw
          if (lane < 31 || (STRIP && !last_strip)) {  // lane 31 of a strip: the halo chunk
#pragma unroll
            for (int v = 0; v < NBV; ++v)
              nbv[v] = *reinterpret_cast<const VT*>(cvec(lane + 1, v));
          }
#pragma unroll
          for (int j = 0; j < M2; ++j) {
#pragma unroll
            for (int r = K2 - 2; r >= 0; --r) a[j * K2 + r] = Op::apply(a[j * K2 + r], a[j * K2 + r + 1]);
            const bool last = (lane == 31) && (j == M2 - 1) && (!STRIP || last_strip);  // n2 % K2 == 0
            if (!last) {
              if (j + 1 < M2) {
                T Pr = a[(j + 1) * K2];
#pragma unroll
                for (int r = 1; r < K2; ++r) {
                  if (r >= 2) Pr = Op::apply(Pr, a[(j + 1) * K2 + r - 1]);
                  a[j * K2 + r] = Op::apply(a[j * K2 + r], Pr);
                }
              } else {
                T Pr = nbv[0].v[0];
#pragma unroll
                for (int r = 1; r < K2; ++r) {
                  if (r >= 2) Pr = Op::apply(Pr, nbv[(r - 1) / VE].v[(r - 1) % VE]);
                  a[j * K2 + r] = Op::apply(a[j * K2 + r], Pr);
                }
              }
            }
          }
          if constexpr (ADD_EXCL) {
            // block heads hold the in-block suffix at the block start = the
            // block total (the stitch never touches block starts): the row
            // total is M2-1 adds and a warp reduction, off the scan chains
            T lt = a[0];
#pragma unroll
            for (int j = 1; j < M2; ++j) lt = Op::apply(lt, a[j * K2]);
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) lt = Op::apply(lt, __shfl_xor_sync(0xffffffffu, lt, d));
            rtot = lt;
          }
          __syncwarp();
          T etail = T(0);
          if constexpr (ADD_EXCL) etail = OpAdd::apply(rtot, tails[ri]);  // row total + tail
#pragma unroll
          for (int v = 0; v < CV; ++v) {
            VT q;
#pragma unroll
            for (int j = 0; j < VE; ++j) {
              const T w = a[v * VE + j];
              if constexpr (ADD_EXCL) {
                q.v[j] = OpAdd::inverse<T>(etail, w);  // (row total + tail) - window
              } else {
                q.v[j] = epi ? OpAdd::inverse<T>(tot, w) : w;
              }
            }
            *reinterpret_cast<VT*>(cvec(lane, v)) = q;
          }
        } else if constexpr (MODE == ROW_EXCL_BLK) {
          // box-complement row round with kx == K2 (the box is cubic in the
          // last two axes) and any monoid: the lane chunk holds M2 whole
          // K2-blocks, and for x at offset r of block j the excluded set
          // [0, x) u [x+K2, n2) is
          //   (blocks left of j) (+) p_j[r-1] (+) s_{j+1}[r] (+) (blocks right of j+1)
          // with p / s the in-block prefix / suffix -- 4 applications per
          // element instead of the full-row P / S chains' 6 (C2 int64 max:
          // each is 2 ISETP + 2 SEL).  Reassociated for floats (tolerance,
          // like ROW_EXCL); exact for max.
          constexpr int NBV = (K2 + VE - 1) / VE;
          T nb[NBV * VE];  // next lane's first block, raw (identity past the row)
#pragma unroll
          for (int v = 0; v < NBV; ++v) {
            VT q;
            if (lane < 31) q = *reinterpret_cast<const VT*>(cvec(lane + 1, v));
#pragma unroll
            for (int j = 0; j < VE; ++j) nb[v * VE + j] = lane < 31 ? q.v[j] : ident;
          }
          T bt[M2];  // block totals
#pragma unroll
          for (int j = 0; j < M2; ++j) {
            T t0 = a[j * K2], t1 = a[j * K2 + 1];
#pragma unroll
            for (int r = 2; r < K2; r += 2) {
              t0 = Op::apply(t0, a[j * K2 + r]);
              if (r + 1 < K2) t1 = Op::apply(t1, a[j * K2 + r + 1]);
            }
            bt[j] = K2 > 1 ? Op::apply(t0, t1) : t0;
          }
          T lt = bt[0];
#pragma unroll
          for (int j = 1; j < M2; ++j) lt = Op::apply(lt, bt[j]);
          // exclusive warp scans of the lane totals
          T pin = lt, sin = lt;
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
          // R[j]: blocks right of block j (in this row)
          T R[M2];
          R[M2 - 1] = suf;
#pragma unroll
          for (int j = M2 - 2; j >= 0; --j) R[j] = Op::apply(bt[j + 1], R[j + 1]);
          // blocks right of the next lane's block 0
          T Rn = __shfl_down_sync(0xffffffffu, R[0], 1);
          if (lane == 31) Rn = ident;
          __syncwarp();
          const T tail = tails[ri];
          T BP = pre;  // blocks left of block j
#pragma unroll
          for (int j = 0; j < M2; ++j) {
            // in-block suffix of block j+1 (own chunk or the next lane's)
            T sn[K2];
            if (j + 1 < M2) {
              sn[K2 - 1] = a[(j + 1) * K2 + K2 - 1];
#pragma unroll
              for (int r = K2 - 2; r >= 0; --r) sn[r] = Op::apply(a[(j + 1) * K2 + r], sn[r + 1]);
            } else {
              sn[K2 - 1] = nb[K2 - 1];
#pragma unroll
              for (int r = K2 - 2; r >= 0; --r) sn[r] = Op::apply(nb[r], sn[r + 1]);
            }
            const T A = Op::apply(Op::apply(BP, j + 1 < M2 ? R[j + 1] : Rn), tail);
            BP = Op::apply(BP, bt[j]);
            T run = A;  // A (+) p_j[r-1]
#pragma unroll
            for (int r = 0; r < K2; ++r) {
              const T raw = a[j * K2 + r];
              a[j * K2 + r] = Op::apply(run, sn[r]);
              run = Op::apply(run, raw);
            }
          }
#pragma unroll
          for (int v = 0; v < CV; ++v) {
            VT q;
#pragma unroll
            for (int j = 0; j < VE; ++j) q.v[j] = a[v * VE + j];
            *reinterpret_cast<VT*>(cvec(lane, v)) = q;
          }
        } else {
          // full-row prefix / suffix.  The lane chunk is cut into SUB
          // sub-chunks whose folds and scans run as independent chains
          // (latency ~C/SUB + log2(32) steps instead of ~3C).
          constexpr int SUB = C >= 16 ? 4 : (C >= 8 ? 2 : 1);
          constexpr int CS = C / SUB;
          T st[SUB];
#pragma unroll
          for (int q = 0; q < SUB; ++q) st[q] = a[q * CS];
#pragma unroll
          for (int j = 1; j < CS; ++j)
#pragma unroll
            for (int q = 0; q < SUB; ++q) st[q] = Op::apply(st[q], a[q * CS + j]);
          T lt = st[0];
#pragma unroll
          for (int q = 1; q < SUB; ++q) lt = Op::apply(lt, st[q]);
          T pin = lt, sin = lt;
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
          // per sub-chunk carries: S enters from the right, P from the left
          T sc[SUB], pc[SUB];
          sc[SUB - 1] = suf;
#pragma unroll
          for (int q = SUB - 2; q >= 0; --q) sc[q] = Op::apply(st[q + 1], sc[q + 1]);
          pc[0] = pre;
#pragma unroll
          for (int q = 1; q < SUB; ++q) pc[q] = Op::apply(pc[q - 1], st[q - 1]);
          {
            // S chains per sub-chunk, written back as 16-byte vectors (a
            // scalar store at the 36-word lane stride would be 4-way conflicted)
            static_assert(CS % VE == 0, "sub-chunks hold whole vectors");
            T run[SUB];
#pragma unroll
            for (int q = 0; q < SUB; ++q) run[q] = sc[q];
#pragma unroll
            for (int jv = CS / VE - 1; jv >= 0; --jv) {
              VT tq[SUB];
#pragma unroll
              for (int j = VE - 1; j >= 0; --j)
#pragma unroll
                for (int q = 0; q < SUB; ++q) {
                  run[q] = Op::apply(a[q * CS + jv * VE + j], run[q]);
                  tq[q].v[j] = run[q];
                }
#pragma unroll
              for (int q = 0; q < SUB; ++q)
                *reinterpret_cast<VT*>(cvec(lane, (q * CS) / VE + jv)) = tq[q];
            }
          }
          __syncwarp();
          T tail = tails[0];
#pragma unroll
          for (int i = 1; i < RPW; ++i)
            if (ri == i) tail = tails[i];
          // out[x] = P[x-1] (+) S[x+k] (+) tail; P runs per sub-chunk from pc[q]
          T pe[SUB];
#pragma unroll
          for (int q = 0; q < SUB; ++q) pe[q] = pc[q];
          if (kvec) {
            // the shift keeps vector alignment: S[x+k] read as 16-byte vectors
#pragma unroll
            for (int v = 0; v < CV; ++v) {
              const int64_t y0 = (int64_t)lane * C + v * VE + kx;
              VT sq;
              if (y0 < N2) {
                if constexpr (SWZ) sq = *reinterpret_cast<const VT*>(wrow + eoff(y0));
                else sq = *reinterpret_cast<const VT*>(wrow + (y0 / C) * CH + (y0 % C));
              } else {
#pragma unroll
                for (int j = 0; j < VE; ++j) sq.v[j] = ident;
              }
#pragma unroll
              for (int j = 0; j < VE; ++j) {
                const int e = v * VE + j;
                const int q = e / CS;
                const T ov = Op::apply(Op::apply(pe[q], sq.v[j]), tail);
                pe[q] = Op::apply(pe[q], a[e]);
                a[e] = ov;
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < C; ++e) {
              const int q = e / CS;
              const int64_t y = (int64_t)lane * C + e + kx;
              T sv = ident;
              if constexpr (SWZ) { if (y < N2) sv = wrow[eoff(y)]; }
              else { if (y < N2) sv = wrow[(y / C) * CH + (y % C)]; }
              const T ov = Op::apply(Op::apply(pe[q], sv), tail);
              pe[q] = Op::apply(pe[q], a[e]);
              a[e] = ov;
            }
          }
          __syncwarp();
#pragma unroll
          for (int v = 0; v < CV; ++v) {
            VT q;
#pragma unroll
            for (int j = 0; j < VE; ++j) q.v[j] = a[v * VE + j];
            *reinterpret_cast<VT*>(cvec(lane, v)) = q;
          }
        }
        __syncwarp();
      }
      __syncthreads();
      if constexpr (DEFER) {
        prev_rows = rows_u;
        prev_us = us;
      } else {
        if (!halo_thr)
          for (int r = 0; r < rows_u; ++r)
            st_stream<T, TV>(dst + (us + r) * rs, *reinterpret_cast<const CT*>(wst + r * ROWP + pcol));
      }
      if constexpr (!EARLY) {
        if (u + 1 < u_end) {
#pragma unroll
          for (int r = 0; r < U; ++r)
            if (r < nlen_u) cur[r] = *reinterpret_cast<const CT*>(sn + r * RAWP);
        }
        issue(u + 3);  // refills the slot unit u+1 just vacated
      }
    }
    if constexpr (DEFER) {
      for (int r = 0; r < (halo_thr ? 0 : prev_rows); ++r)
        st_stream<T, TV>(dst + (prev_us + r) * rs, *reinterpret_cast<const CT*>(wst + r * ROWP + pcol));
    }
    cp_async_wait<0>();
  }
}

// threads own TV-element column vectors: ~256-512 threads per CTA
template <class T, int C>
constexpr int pick_tv() {
  return (32 * C) / (16 / (int)sizeof(T)) >= 256 ? ((32 * C) / 512 >= 1 ? (32 * C) / 512 : 1)
                                                 : (32 * C) / 256 >= 1 ? (32 * C) / 256 : 1;
}

template <class T, class Op, int C, int K1, int MODE, bool STRIP>
int go_pair(const T* in, T* out, int64_t outer, int64_t n1, int64_t kx,
            const typename AccOf<T>::type* total, const T* Tail, int64_t n2full, cudaStream_t s) {
  constexpr int VE = 16 / sizeof(T);
  constexpr int TV = VE;  // 16-byte column vectors measured best (8-byte: -30% at C4)
  constexpr int N2 = 32 * C;
  constexpr int NT = N2 / TV;
  constexpr int CV = C / VE;
  constexpr int HV = STRIP ? (K1 - 1 + VE - 1) / VE : 0;
  constexpr int ROWP = (STRIP ? 33 : 32) * fp_chunk_stride(CV, MODE, STRIP) * VE;
  constexpr int U = fp_unit_rows(C, K1);
  constexpr int NTA = NT + (STRIP ? 32 : 0);
  const int64_t nstrips = STRIP ? n2full / N2 : 1;
  const size_t smem = ((size_t)2 * U * (N2 + HV * VE) + (size_t)U * ROWP) * sizeof(T);
  if (smem > 220 * 1024) return -1;
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm > 2048 / NTA) per_sm = 2048 / NTA;
  if (per_sm < 1) per_sm = 1;
  const int64_t nunits = (n1 + U - 1) / U;
  // segments per outer index (exsum_launch.h: wave rounding vs halo + fill)
  int64_t nseg = pick_segments(outer * nstrips, nunits, per_sm);
  int64_t seg_len = U * ((nunits + nseg - 1) / nseg);
  nseg = (n1 + seg_len - 1) / seg_len;
  const int64_t items = outer * nseg * nstrips;
  int64_t grid = items;
  const int64_t cap = (int64_t)num_sms() * per_sm * 4;
  if (grid > cap) grid = cap;
  // one resident CTA per SM and few lines: when the best uniform segmentation
  // still costs FP_BALANCED_PCT % more than an even split of the units (a
  // partial last wave, or a halo block per short segment), cut the units
  // into one contiguous range per SM instead (balanced ranges of the kernel).
  // The windowed row op with a small window measured slower that way; with
  // more lines than SMs it keeps whole-line items for the full waves of lines
  // and balances only the last partial wave (FP_BALANCED_TAIL)
  const int bal_mode = fp_balanced_mode();
  int64_t bal_line0 = 0;
  int bal_ctas = 0;
  if ((!STRIP || FP_BALANCED_STRIPS) && per_sm == 1 && bal_mode) {
    const int64_t slots = num_sms();
    const int64_t lines = outer * nstrips;
    const int64_t per = seg_len / U;
    const double uniform = (double)((items + slots - 1) / slots) * ((double)per + 1.0);
    const double even = (double)(lines * nunits) / (double)slots + 2.0;
    const bool pays = bal_mode == 2 || (lines * nunits >= 4 * slots &&
                                        uniform * 100.0 > even * (100.0 + FP_BALANCED_PCT));
    const bool small_win = MODE == ROW_WIN && K1 < FP_BALANCED_MIN_K_WIN;
    if (pays && (!small_win || bal_mode == 2)) {
      bal_ctas = (int)(slots * FP_BALANCED_MULT);
      grid = bal_ctas;
    } else if (pays && FP_BALANCED_TAIL && lines > slots && lines % slots != 0) {
      bal_line0 = (lines / slots) * slots;
      bal_ctas = (int)slots;
      nseg = 1;
      seg_len = U * nunits;
      grid = bal_line0 + bal_ctas;  // one whole line per CTA, then the ranges
    }
  }
  ensure_smem((const void*)k_fused_pair<T, Op, C, K1, MODE, TV, STRIP>, smem);
  k_fused_pair<T, Op, C, K1, MODE, TV, STRIP><<<(unsigned)grid, NTA, smem, s>>>(
      in, out, outer, n1, kx, seg_len, nseg, total, Tail, STRIP ? n2full : (int64_t)N2, nstrips,
      bal_line0, bal_ctas);
  return 1;
}

template <class T, class Op, int C, int MODE, bool STRIP = false>
int pick_k1(const T* in, T* out, int64_t outer, int64_t n1, int64_t k1, int64_t kx,
            const typename AccOf<T>::type* total, const T* Tail, cudaStream_t s,
            int64_t n2full = 0) {
  switch (k1) {
    case 2: return go_pair<T, Op, C, 2, MODE, STRIP>(in, out, outer, n1, kx, total, Tail, n2full, s);
    case 4: return go_pair<T, Op, C, 4, MODE, STRIP>(in, out, outer, n1, kx, total, Tail, n2full, s);
    case 8: return go_pair<T, Op, C, 8, MODE, STRIP>(in, out, outer, n1, kx, total, Tail, n2full, s);
    case 16:
      if constexpr (C >= 16)
        return go_pair<T, Op, C, 16, MODE, STRIP>(in, out, outer, n1, kx, total, Tail, n2full, s);
      return -1;
  }
  return -1;
}

template <class T, class Op>
int go_fused(const T* in, T* out, int64_t outer, int64_t n1, int64_t n2, int64_t k1, int64_t k2,
             int mode, const typename AccOf<T>::type* total, const T* Tail, cudaStream_t s) {
  if (((uintptr_t)in % 16) || ((uintptr_t)out % 16)) return -1;
  if (mode == ROW_WIN) {
    // rows longer than the widest row template: strips of it with a halo
    constexpr int CW = sizeof(T) == 4 ? 32 : 16;
    // small windows on rows longer than the widest template: 256-column strips
    // (4-8-row units, a 25-50 KB ring and stage: 4 CTAs per SM instead of one
    // 200 KB CTA of 9 warps).  Measured (tools/variant_time.py): 8-byte 4096^2
    // box 4^2 max 75.8 -> 61.4 us, + 71.7 -> 57.3 us, box 8^2 max 90.6 -> 74.2
    // us; float32 only for k = 2 (64x2048x2048 box 2^3 pair 0.404 -> 0.361 ms;
    // 4096^2 box 4^2 34.8 -> 36.9 us and box 8^2 35 -> 59 us stay on 1024-wide strips)
    if (n2 > 32 * CW && n2 % 256 == 0 && k1 <= (sizeof(T) == 8 ? FP_STRIP_NARROW_K8 : FP_STRIP_NARROW_K4))
      return pick_k1<T, Op, 8, ROW_WIN, true>(in, out, outer, n1, k1, 0, total, nullptr, s, n2);
    if (n2 > 32 * CW && n2 % (32 * CW) == 0)
      return pick_k1<T, Op, CW, ROW_WIN, true>(in, out, outer, n1, k1, 0, total, nullptr, s, n2);
    switch (n2) {
      case 256: return pick_k1<T, Op, 8, ROW_WIN>(in, out, outer, n1, k1, 0, total, nullptr, s);
      case 512: return pick_k1<T, Op, 16, ROW_WIN>(in, out, outer, n1, k1, 0, total, nullptr, s);
      case 1024:
        if constexpr (sizeof(T) == 4) return pick_k1<T, Op, 32, ROW_WIN>(in, out, outer, n1, k1, 0, total, nullptr, s);
        return -1;
    }
  } else {
    // integer + with a cubic box: row total minus the exact windowed row op
    // (two's-complement wrap makes the inverse exact; 8-byte elements for
    // k <= 4 or 256-wide rows: larger windows on wider rows spill; C2 int64
    // box-complement fused pass 0.084 -> 0.060 ms).  Floats never take it:
    // box-complement is the strong route, no subtraction anywhere
    // (excluded.py:130) -- they take ROW_EXCL_BLK below.
    if constexpr (std::is_same<Op, OpAdd>::value && std::is_integral<T>::value) {
      if (k2 == k1 && (sizeof(T) == 4 || k1 <= 4 || n2 == 256)) {
        switch (n2) {
          case 256: return pick_k1<T, Op, 8, ROW_EXCL_ADD>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
          case 512: return pick_k1<T, Op, 16, ROW_EXCL_ADD>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
          case 1024:
            if constexpr (sizeof(T) == 4) return pick_k1<T, Op, 32, ROW_EXCL_ADD>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
            return -1;
        }
      }
    }
    // cubic in the last two axes: the block-decomposed row round (any monoid)
    if (k2 == k1 && FP_EXCL_BLK) {
      switch (n2) {
        case 256: return pick_k1<T, Op, 8, ROW_EXCL_BLK>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
        case 512: return pick_k1<T, Op, 16, ROW_EXCL_BLK>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
        case 1024:
          if constexpr (sizeof(T) == 4) return pick_k1<T, Op, 32, ROW_EXCL_BLK>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
          return -1;
      }
    }
    switch (n2) {
      case 256: return pick_k1<T, Op, 8, ROW_EXCL>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
      case 512: return pick_k1<T, Op, 16, ROW_EXCL>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
      case 1024:
        if constexpr (sizeof(T) == 4) return pick_k1<T, Op, 32, ROW_EXCL>(in, out, outer, n1, k1, k2, nullptr, Tail, s);
        return -1;
    }
  }
  return -1;
}

}  // namespace exsum
