// axis_stream.cuh -- strided windowed pass through a cp.async shared ring.
//
// Same algorithm and association as windowed_sum_axis (reference
// pkg/src/exsum/scan.py:61-102) on a view [outer, n, inner]: in-block
// right-nested suffix, left-nested prefix of the next block, one stitch
// combine.  The B200 mapping is the streaming half of fused_pair.cuh: a CTA
// owns a strip of N2 = 32*C consecutive columns of one outer index and a
// segment of the axis; every thread owns one 16-byte column vector and
// prefetches its own vectors of units u+2, u+3 (U = 16 rows) with cp.async
// into a 2-slot ring, the suffix/prefix run in registers, results go straight
// to HBM as coalesced 16-byte stores.
//
// Piggy-backed reductions of the raw input (the pass reads it anyway):
//   EX == 1: R, the fold of every row of the last axis (box-complement,
//            exsum_capi.cu): each thread folds its 16-byte vector of every
//            row of the unit, a 16-value warp butterfly (17 shuffles) folds
//            those across the warp's 128 columns, one partial per (row,
//            128-column segment) -- no CTA barrier (a shared-memory fold
//            needed two per unit and ran at 1.96 ms vs 1.42 ms on C4).  The
//            butterfly of unit u+1 runs on its raw registers during unit u
//            (AS_FOLD_NEXT), so its shuffle latency overlaps the block
//            compute: C4 pass 1.426 -> 1.403 ms;
//   EX == 2: the BDBSC total, folded per thread from registers.
#pragma once

#include <stdlib.h>

#include <type_traits>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

#ifndef AS_RING
#define AS_RING 2  // shared-memory ring slots (units in flight beyond the two in registers)
#endif
#ifndef AS_ABL
#define AS_ABL 0  // measurement only: 1 skips the row-partial stores, 2 the whole fold
#endif
#ifndef AS_DEFER
#define AS_DEFER 0  // 1: unit u's output rows leave during unit u+1 through a per-thread stage
#endif
#ifndef AS_GRID_MULT
#define AS_GRID_MULT 4  // grid cap in resident CTAs (items are grid-strided)
#endif
#ifndef AS_PSTRIDE
#define AS_PSTRIDE 1  // measurement only: strip order multiplier (must be coprime to the strip count)
#endif
#ifndef AS_NSEG_MIN
#define AS_NSEG_MIN 1  // measurement only: at least this many axis segments
#endif
#ifndef AS_SEG_FAST
#define AS_SEG_FAST 0  // measurement only: 1 makes the segment the fastest item index
#endif
#ifndef AS_NO_C32
#define AS_NO_C32 0  // measurement only: 1 keeps 4-byte types on the 512-column strip
#endif

// the last partial wave of whole-line items as balanced unit ranges (see the
// kernel); AS_BAL_GU_MULT > 0 caps the CTAs of the uniform part at that many
// per SM (grid-strided) instead of one CTA per line; EXSUM_AS_BAL_TAIL=0: off
#ifndef AS_BAL_TAIL
#define AS_BAL_TAIL 1
#endif
#ifndef AS_BAL_GU_MULT
#define AS_BAL_GU_MULT 0
#endif
// EXSUM_AS_BAL_TAIL: 0 off, 1 (default) where whole-line items were chosen,
// 2 whole-line items and a balanced last wave whenever the lines allow it (tests)
inline int as_bal_tail_mode() {
  const char* e = getenv("EXSUM_AS_BAL_TAIL");
  return e && e[0] >= '0' && e[0] <= '2' ? e[0] - '0' : 1;
}

template <class T, class Op, int C, int K1, int EX>
__global__ void __launch_bounds__(32 * C / (16 / sizeof(T)), 1)
k_axis_stream(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n1,
              int64_t inner, int64_t nout, int64_t seg_len, int64_t nseg,
              const typename AccOf<T>::type* __restrict__ total, T* __restrict__ rowpart,
              int64_t row_len, typename AccOf<T>::type* __restrict__ tpart, int64_t bal_line0,
              int bal_ctas) {
  typedef typename AccOf<T>::type Acc;
  constexpr int VE = 16 / sizeof(T);
  constexpr int N2 = 32 * C;                     // strip width (columns)
  constexpr int NT = N2 / VE;                    // threads
  constexpr int NW = NT / 32;
  constexpr int G = 16 / K1 > 0 ? 16 / K1 : 1;   // blocks per unit
  constexpr int U = G * K1;                      // rows per unit
  typedef Vec<T, VE> VT;
  extern __shared__ __align__(16) unsigned char smem[];
  T* raw = reinterpret_cast<T*>(smem);  // [AS_RING][U][N2]
  // AS_DEFER: a stage of U output rows; each thread touches only its own
  // column vector of it, so no barrier is needed
  T* stg = raw + AS_RING * U * N2;      // [U][N2]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int col = tid * VE;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t last_bs = (int64_t)K1 * ((n1 - 1) / K1);
  const int64_t strips = inner / N2;
  const int64_t items = outer * strips * nseg;
  Acc tacc[VE];
#pragma unroll
  for (int j = 0; j < VE; ++j) tacc[j] = Op::template identity<Acc>();

  // Balanced tail (bal_ctas > 0; whole-line items, nseg == 1): the lines
  // [0, bal_line0) -- whole waves of one line per SM -- run as uniform items
  // on the first gridDim.x - bal_ctas CTAs; the units of the remaining lines
  // (less than one wave of lines) are cut into bal_ctas equal contiguous
  // ranges, one per CTA, so the last wave ends together instead of leaving
  // the SMs without a line idle for a whole item.
  const int64_t gu = (int64_t)gridDim.x - bal_ctas;
  const bool bal = bal_ctas > 0 && (int64_t)blockIdx.x >= gu;
  const int64_t nun = (nout + U - 1) / U;  // units per line
  const int64_t tail_units = (outer * strips - bal_line0) * nun;
  int64_t item = bal ? tail_units * ((int64_t)blockIdx.x - gu) / bal_ctas : (int64_t)blockIdx.x;
  const int64_t item_end = bal ? tail_units * ((int64_t)blockIdx.x - gu + 1) / bal_ctas
                               : (bal_ctas > 0 ? bal_line0 : items);
  while (item < item_end) {
    int64_t strip, o, xs, xe;
    if (bal) {
      const int64_t l = item / nun, us = item - l * nun;
      const int64_t cnt = nun - us < item_end - item ? nun - us : item_end - item;
      strip = (bal_line0 + l) % strips;
      o = (bal_line0 + l) / strips;
      xs = us * U;
      xe = (us + cnt) * U < nout ? (us + cnt) * U : nout;
      item += cnt;
    } else {
      const int64_t it2 = AS_SEG_FAST ? (item % nseg) * (outer * strips) + item / nseg : item;
      strip = AS_PSTRIDE == 1 ? it2 % strips : (it2 % strips) * AS_PSTRIDE % strips;
      const int64_t rest = it2 / strips;
      o = rest % outer;
      const int64_t seg = rest / outer;
      xs = seg * seg_len;  // multiple of U
      xe = xs + seg_len < nout ? xs + seg_len : nout;
      item += gu;
    }
    const int64_t u0 = xs / U;
    const int64_t u_end = (xe + U - 1) / U;
    const T* src = in + o * n1 * inner + strip * N2 + col;
    T* dst = out + o * nout * inner + strip * N2 + col;
    // EX == 1: where this warp's row partials go -- rowpart[row][seg] with
    // row = (o * nout + x) * rpi + cq / row_len, seg = (cq % row_len) / 128
    // (inner is a multiple of row_len): a row's partials are contiguous, so the
    // CTA's warps fill whole lines together (a [seg][row] layout scattered them
    // over row_len / 128 regions: C4 pass 1.409 -> see DESIGN); the divisions
    // once per item, not per unit
    int64_t rp_base = 0, rp_step = 0;
    if constexpr (EX == 1) {
      const int64_t cq = strip * N2 + warp * (32 * VE);
      const int64_t ppr = row_len / (32 * VE);
      rp_step = (inner / row_len) * ppr;
      rp_base = (o * nout * (inner / row_len) + cq / row_len) * ppr + (cq % row_len) / (32 * VE);
    }

    auto rows_of = [&](int64_t ui) -> int {
      const int64_t avail = n1 - ui * U;
      const int64_t want = ui >= u_end ? K1 - 1 : U;
      return (int)(avail < want ? (avail > 0 ? avail : 0) : want);
    };
    auto issue = [&](int64_t ui) {
      const int rows = rows_of(ui);
      T* d = raw + ((ui - u0) % AS_RING) * (U * N2) + col;
      for (int r = 0; r < rows; ++r) cp_async16(d + r * N2, src + (ui * U + r) * inner);
      cp_async_commit();
    };
    // EX == 1: fold the unit's own raw rows across the warp (32 lanes x 4
    // columns = 128 columns of a row) with a multi-value butterfly: 15+2
    // shuffles for 16 rows; lanes whose low bits are zero store one partial
    // per (row, 128-column segment) to rowpart[segment][row].
    auto fold_rows = [&](const VT (&blk)[U], int64_t x0, int nrows) {
      if constexpr (EX == 1 && AS_ABL != 2) {
        T sv[U];
#pragma unroll
        for (int r = 0; r < U; ++r) {
          T sum = blk[r].v[0];
#pragma unroll
          for (int j = 1; j < VE; ++j) sum = Op::apply(sum, blk[r].v[j]);
          sv[r] = r < nrows ? sum : Op::template identity<T>();
        }
        int rowbase = 0;
#pragma unroll
        for (int cnt = U, off = 16; cnt > 1; cnt >>= 1, off >>= 1) {
          const int half = cnt >> 1;
          const bool hi = (lane & off) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const T send = hi ? sv[i] : sv[i + half];
            const T keep = hi ? sv[i + half] : sv[i];
            sv[i] = Op::apply(keep, __shfl_xor_sync(0xffffffffu, send, off));
          }
          rowbase += hi ? half : 0;
        }
        constexpr int LOWB = 32 / U;
#pragma unroll
        for (int off = LOWB >> 1; off >= 1; off >>= 1)
          sv[0] = Op::apply(sv[0], __shfl_xor_sync(0xffffffffu, sv[0], off));
        if (AS_ABL == 1 && sv[0] != T(-12345.678)) return;
        if ((lane & (LOWB - 1)) == 0 && rowbase < nrows) {
          rowpart[rp_base + (x0 + rowbase) * rp_step] = sv[0];
        }
      }
    };

#pragma unroll
    for (int i = 0; i < AS_RING; ++i) issue(u0 + i);
    cp_async_wait<AS_RING - 1>();
    VT cur[U];
    int len = rows_of(u0);
#pragma unroll
    for (int r = 0; r < U; ++r)
      if (r < len) cur[r] = *reinterpret_cast<const VT*>(raw + col + r * N2);
    issue(u0 + AS_RING);

    [[maybe_unused]] int prev_w = 0;  // AS_DEFER: stage rows [0, prev_w) still hold unit prev_us's output
    [[maybe_unused]] int64_t prev_us = 0;
    auto flush = [&](int from, int to) {
      for (int r = from; r < to; ++r)
        st_stream<T, VE>(dst + (prev_us + r) * inner, *reinterpret_cast<const VT*>(stg + r * N2 + col));
    };

    for (int64_t u = u0; u < u_end; ++u) {
      const int64_t us = u * U;
      const int rows_u = len;
#ifndef AS_FOLD_NEXT
#define AS_FOLD_NEXT 1
#endif
      if (!AS_FOLD_NEXT || u == u0) {
        const int64_t inseg = xe - us;
        fold_rows(cur, us, (int)(rows_u < inseg ? rows_u : inseg));
      }
      if constexpr (EX == 2) {
#pragma unroll
        for (int r = 0; r < U; ++r)
          if (r < rows_u && us + r < xe) {
#pragma unroll
            for (int j = 0; j < VE; ++j) tacc[j] = Op::apply(tacc[j], (Acc)cur[r].v[j]);
          }
      }
      const int nlen_u = rows_of(u + 1);
      const T* sn = raw + ((u + 1 - u0) % AS_RING) * (U * N2) + col;
      VT nxt[U];
      if (nlen_u > 0) {
        cp_async_wait<AS_RING - 1>();  // unit u+1 has landed (u+2.. may still be in flight)
#pragma unroll
        for (int r = 0; r < U; ++r)
          if (r < nlen_u) nxt[r] = *reinterpret_cast<const VT*>(sn + r * N2);
      }
      issue(u + AS_RING + 1);
      if (AS_FOLD_NEXT && u + 1 < u_end) {
        // the next unit's row partials now, from its raw registers: the
        // butterfly's shuffle latency overlaps this unit's block compute
        const int64_t usn = us + U;
        const int64_t inseg = xe - usn;
        fold_rows(nxt, usn, (int)(nlen_u < inseg ? nlen_u : inseg));
      }
#pragma unroll
      for (int jb = 0; jb < G; ++jb) {
        const int64_t bs = us + (int64_t)jb * K1;
        if (jb * K1 < rows_u && bs < xe) {  // the unit may reach into a shard's halo
          const int blen = (int)(n1 - bs < K1 ? n1 - bs : K1);
#pragma unroll
          for (int r = K1 - 2; r >= 0; --r)
            if (r < blen - 1) {
#pragma unroll
              for (int j = 0; j < VE; ++j)
                cur[jb * K1 + r].v[j] = Op::apply(cur[jb * K1 + r].v[j], cur[jb * K1 + r + 1].v[j]);
            }
          auto put = [&](int r, VT w) {
            if (epi) {
#pragma unroll
              for (int j = 0; j < VE; ++j) w.v[j] = OpAdd::inverse<T>(tot, w.v[j]);
            }
            if constexpr (AS_DEFER) {
              const int slot = jb * K1 + r;
              VT* sp = reinterpret_cast<VT*>(stg + slot * N2 + col);
              if (slot < prev_w) st_stream<T, VE>(dst + (prev_us + slot) * inner, *sp);
              *sp = w;
            } else {
              st_stream<T, VE>(dst + (bs + r) * inner, w);
            }
          };
          if (bs == last_bs) {
#pragma unroll
            for (int r = 0; r < K1; ++r)
              if (r < blen) put(r, cur[jb * K1 + r]);
          } else {
            const int64_t nrows = n1 - bs - K1;
            const int nlen = (int)(nrows < K1 ? nrows : K1);
            put(0, cur[jb * K1]);
            const int nb0 = jb + 1 < G ? (jb + 1) * K1 : 0;
            VT P = jb + 1 < G ? cur[nb0] : nxt[0];
#pragma unroll
            for (int r = 1; r < K1; ++r) {
              const int jj = r - 1;
              if (jj >= 1 && jj < nlen) {
                const VT av = jb + 1 < G ? cur[nb0 + jj] : nxt[jj];
#pragma unroll
                for (int j = 0; j < VE; ++j) P.v[j] = Op::apply(P.v[j], av.v[j]);
              }
              VT w;
#pragma unroll
              for (int j = 0; j < VE; ++j) w.v[j] = Op::apply(cur[jb * K1 + r].v[j], P.v[j]);
              put(r, w);
            }
          }
        }
      }
      if constexpr (AS_DEFER) {
        // this unit wrote stage rows [0, w): the rest of the previous unit's leave now
        const int64_t wr = (xe - us < rows_u ? xe - us : rows_u);
        const int w = (int)(wr > 0 ? wr : 0);
        flush(w, prev_w);
        prev_w = w;
        prev_us = us;
      }
      len = nlen_u;
      if (u + 1 < u_end) {
#pragma unroll
        for (int r = 0; r < U; ++r) cur[r] = nxt[r];
      }
    }
    if constexpr (AS_DEFER) flush(0, prev_w);
    cp_async_wait<0>();
    __syncthreads();  // the next item refills both slots
  }
  if constexpr (EX == 2) {
    __shared__ Acc sh[NW];
    Acc ta = tacc[0];
#pragma unroll
    for (int j = 1; j < VE; ++j) ta = Op::apply(ta, tacc[j]);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) ta = Op::apply(ta, __shfl_xor_sync(0xffffffffu, ta, d));
    if (lane == 0) sh[warp] = ta;
    __syncthreads();
    if (tid == 0) {
      Acc t = sh[0];
      for (int w = 1; w < NW; ++w) t = Op::apply(t, sh[w]);
      tpart[blockIdx.x] = t;
    }
  }
}

// ---- host dispatch (instantiated once per element type / operator in
// axis_stream_{f32,f64,i64add,i64max}.cu so they compile in parallel) ----

template <class T, class Op, int C, int K1, int EX>
int go_axis_stream_c(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t nout,
                     const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  typedef typename AccOf<T>::type Acc;
  constexpr int VE = 16 / sizeof(T);
  constexpr int N2 = 32 * C;
  constexpr int NT = N2 / VE;
  constexpr int U = (16 / K1) * K1;
  const size_t smem = (size_t)(AS_RING + (AS_DEFER ? 1 : 0)) * U * N2 * sizeof(T);
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm > 2048 / NT) per_sm = 2048 / NT;
  if (per_sm < 1) per_sm = 1;
  const int64_t strips = inner / N2;
  const int64_t lines = outer * strips;
  const int64_t nunits = (nout + U - 1) / U;
  int64_t nseg = pick_segments(lines, nunits, per_sm);
  if (nseg < AS_NSEG_MIN && nunits >= AS_NSEG_MIN) nseg = AS_NSEG_MIN;
  const int bal_mode = AS_BAL_TAIL ? as_bal_tail_mode() : 0;
  const int64_t slots = (int64_t)num_sms() * per_sm;
  const bool bal_shape = per_sm == 1 && EX != 2 && AS_SEG_FAST == 0 && AS_PSTRIDE == 1 &&
                         lines > slots && lines % slots != 0;
  if (bal_mode == 2 && bal_shape) nseg = 1;
  const int64_t seg_len = U * ((nunits + nseg - 1) / nseg);
  nseg = (nout + seg_len - 1) / seg_len;
  const int64_t items = lines * nseg;
  int64_t grid = items;
  const int64_t cap = (int64_t)num_sms() * per_sm * AS_GRID_MULT;
  if (EX == 2 && cap > ex->cap) return -1;
  if (grid > cap) grid = cap;
  // whole-line items on one resident CTA per SM whose count is not a multiple
  // of the SM count: the last partial wave of lines as balanced unit ranges
  int64_t bal_line0 = 0;
  int bal_ctas = 0;
  if (bal_mode && bal_shape && nseg == 1 && (nunits >= 8 || bal_mode == 2)) {
    bal_line0 = (lines / slots) * slots;
    bal_ctas = (int)slots;
    grid = (AS_BAL_GU_MULT > 0 && bal_line0 > slots * AS_BAL_GU_MULT ? slots * AS_BAL_GU_MULT
                                                                       : bal_line0) + bal_ctas;
  }
  ensure_smem((const void*)k_axis_stream<T, Op, C, K1, EX>, smem);
  k_axis_stream<T, Op, C, K1, EX><<<(unsigned)grid, NT, smem, s>>>(
      in, out, outer, n, inner, nout, seg_len, nseg, total,
      EX == 1 ? (T*)ex->buf : nullptr, EX == 1 ? ex->row_len : N2,
      EX == 2 ? (Acc*)ex->buf : nullptr, bal_line0, bal_ctas);
  if (ex) {
    ex->n_out_done = 1;
    if (EX == 1) {
      ex->done = 1;
      ex->ppr = ex->row_len / (32 * VE);
    } else if (EX == 2) {
      ex->done = 1;
      ex->ppr = grid;
    }
  }
  return 1;
}

template <class T, class Op, int C, int EX>
int pick_axis_k(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t nout,
                int64_t k, const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  switch (k) {
    case 2: return go_axis_stream_c<T, Op, C, 2, EX>(in, out, outer, n, inner, nout, total, s, ex);
    case 4: return go_axis_stream_c<T, Op, C, 4, EX>(in, out, outer, n, inner, nout, total, s, ex);
    case 8: return go_axis_stream_c<T, Op, C, 8, EX>(in, out, outer, n, inner, nout, total, s, ex);
    case 16: return go_axis_stream_c<T, Op, C, 16, EX>(in, out, outer, n, inner, nout, total, s, ex);
  }
  return -1;
}

template <class T, class Op, int C>
int pick_axis_ex(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t nout,
                 int64_t k, const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  const int kind = ex ? ex->kind : 0;
  if (kind == 1) {
    if (ex->row_len % (32 * 16 / (int)sizeof(T)) != 0 || ex->row_len % (32 * C) != 0 ||
        inner % ex->row_len != 0)
      return -1;
    return pick_axis_k<T, Op, C, 1>(in, out, outer, n, inner, nout, k, total, s, ex);
  }
  if constexpr (!std::is_same<Op, OpMax>::value) {
    if (kind == 2) return pick_axis_k<T, Op, C, 2>(in, out, outer, n, inner, nout, k, total, s, ex);
  }
  if (kind != 0) return -1;
  return pick_axis_k<T, Op, C, 0>(in, out, outer, n, inner, nout, k, total, s, ex);
}

template <class T, class Op>
int go_axis_stream(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t k,
                   const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  if (((uintptr_t)in % 16) || ((uintptr_t)out % 16)) return -1;
  if (!(k == 2 || k == 4 || k == 8 || k == 16)) return -1;
  if (n < 64) return -1;  // < 4 units per strip: the ring never fills; register streaming wins
  const int64_t nout = (ex && ex->n_out >= 0) ? ex->n_out : n;
  if (nout != n && outer != 1) return -1;
  if constexpr (sizeof(T) == 4) {
    if (!AS_NO_C32 && inner % 1024 == 0 && (!ex || ex->kind != 1 || ex->row_len % 1024 == 0))
      return pick_axis_ex<T, Op, 32>(in, out, outer, n, inner, nout, k, total, s, ex);
  }
  if (inner % 512 == 0 && (!ex || ex->kind != 1 || ex->row_len % 512 == 0))
    return pick_axis_ex<T, Op, 16>(in, out, outer, n, inner, nout, k, total, s, ex);
  if (inner % 256 == 0 && (!ex || ex->kind != 1 || ex->row_len % 256 == 0))
    return pick_axis_ex<T, Op, 8>(in, out, outer, n, inner, nout, k, total, s, ex);
  return -1;
}

}  // namespace exsum
