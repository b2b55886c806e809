// pass_bulk.cu -- strided windowed pass for large windows, TMA bulk-copy pipeline.
//
// Same algorithm and association as windowed_sum_axis (reference
// pkg/src/exsum/scan.py:61-102): in-block right-nested suffix S, left-nested
// prefix P of the next block, out = S (+) P.
//
// Why a separate kernel: with k > 16 (8-byte) or k > 32 (4-byte) a thread can
// no longer hold a block's suffixes plus the next block in registers
// (register streaming hits 170+ registers and 12% occupancy).  Here each warp
// owns a 32-column strip (lane = column, one 128/256-byte row segment per
// row) and streams its blocks through a ring of R shared-memory stages filled
// by cp.async.bulk (1-D TMA, one copy per row segment, completion on an
// mbarrier with expect_tx).  The suffix runs in place in shared memory, the
// next block's prefix streams from its stage, and results go straight to
// global memory (32 lanes x 8 bytes = one coalesced row per store).  Registers
// are O(1) in k; the ring keeps R-1 blocks of loads in flight per warp.
#include <stdlib.h>

#include <type_traits>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

template <class T, class Op, bool TOT>
__global__ void __launch_bounds__(32)
k_strided_bulk(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n,
               int64_t inner, int k, int64_t seg_len, int64_t nseg, int R,
               const typename AccOf<T>::type* __restrict__ total,
               typename AccOf<T>::type* __restrict__ tpart) {
  // tpart (BDBSC, excluded.py:72-75): this CTA's fold of the raw input rows it
  // owns (the in-block suffix loops read each own row once), for
  // launch_total_final -- the total rides on this pass instead of a separate
  // read of the array
  typedef typename AccOf<T>::type Acc;
  Acc tacc = Acc(0);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // R <= 15 barriers
  T* stg = reinterpret_cast<T*>(smem + 128);
  const int lane = threadIdx.x;
  const int64_t stage_elems = (int64_t)k * 32;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t last_bs = (int64_t)k * ((n - 1) / k);
  const int64_t nb_total = (n + k - 1) / k;
  const int64_t strips = inner / 32;
  const int64_t items = strips * outer * nseg;
  if (lane == 0) {
    for (int i = 0; i < R; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t nload = 0, ncons = 0;  // running load / consume counters -> stage, parity

  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t strip = item % strips;
    const int64_t rest = item / strips;
    const int64_t o = rest % outer;
    const int64_t seg = rest / outer;
    const int64_t xs = seg * seg_len;
    const int64_t xe = xs + seg_len < n ? xs + seg_len : n;
    const int64_t b0 = xs / k;
    const int64_t b_end = (xe + k - 1) / k;
    const int64_t halo = b_end < nb_total ? 1 : 0;
    const int64_t nblk = (b_end - b0) + halo;
    const T* src = in + o * n * inner + strip * 32;
    T* dst = out + o * n * inner + strip * 32 + lane;

    auto rows_of = [&](int64_t bi) -> int {
      const int64_t avail = n - bi * k;
      const int64_t want = bi == b_end ? k - 1 : k;  // the halo needs k-1 rows
      return (int)(avail < want ? avail : want);
    };
    auto issue = [&](int64_t bi) {
      const uint32_t st = nload % R;
      const int rows = rows_of(bi);
      fence_proxy_async_smem();  // generic-proxy writes to the stage happen before the copy
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&bar[st], (uint32_t)(rows * 32 * sizeof(T)));
      __syncwarp();
      T* d = stg + st * stage_elems;
      for (int r = lane; r < rows; r += 32)
        bulk_g2s(d + r * 32, src + (bi * k + r) * inner, 32 * sizeof(T), &bar[st]);
      ++nload;
    };
    auto wait_idx = [&](uint32_t c) { mbar_wait(&bar[c % R], (c / R) & 1); };

    int64_t next_issue = b0;
    for (; next_issue < b0 + nblk && next_issue < b0 + R; ++next_issue) issue(next_issue);

    uint32_t cb = ncons;
    wait_idx(cb);
    T* cur = stg + (cb % R) * stage_elems;
    int len = rows_of(b0);
    {  // in-block suffix of the first block, in place (right nested)
      T v = cur[(len - 1) * 32 + lane];
      if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)v);
#pragma unroll 8
      for (int r = len - 2; r >= 0; --r) {
        const T a = cur[r * 32 + lane];
        if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)a);
        v = Op::apply(a, v);
        cur[r * 32 + lane] = v;
      }
    }
    for (int64_t b = b0; b < b_end; ++b) {
      const int64_t bs = b * k;
      if (bs == last_bs) {  // last block: out = S
        for (int r = 0; r < len; ++r) {
          const T v = cur[r * 32 + lane];
          st1(dst + (bs + r) * inner, epi ? OpAdd::inverse<T>(tot, v) : v);
        }
        break;
      }
      wait_idx(cb + 1);
      T* nxt = stg + ((cb + 1) % R) * stage_elems;
      const int nlen = rows_of(b + 1);
      {
        const T v = cur[lane];
        st1(dst + bs * inner, epi ? OpAdd::inverse<T>(tot, v) : v);
      }
      T P = nxt[lane];
#pragma unroll 8
      for (int r = 1; r < k; ++r) {
        const int jj = r - 1;
        if (jj >= 1 && jj < nlen) P = Op::apply(P, nxt[jj * 32 + lane]);
        const T v = Op::apply(cur[r * 32 + lane], P);
        st1(dst + (bs + r) * inner, epi ? OpAdd::inverse<T>(tot, v) : v);
      }
      // the current stage is free: refill it with the next block in line
      if (next_issue < b0 + nblk) issue(next_issue++);
      ++cb;
      if (b + 1 < b_end) {
        cur = nxt;
        len = nlen;
        T v = cur[(len - 1) * 32 + lane];
        if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)v);
#pragma unroll 8
        for (int r = len - 2; r >= 0; --r) {
          const T a = cur[r * 32 + lane];
          if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)a);
          v = Op::apply(a, v);
          cur[r * 32 + lane] = v;
        }
      }
    }
    ncons += (uint32_t)nblk;
    __syncwarp();
  }
  if constexpr (TOT) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) tacc = OpAdd::apply<Acc>(tacc, __shfl_xor_sync(0xffffffffu, tacc, d));
    if (lane == 0) tpart[blockIdx.x] = tacc;
  }
}

namespace {

template <class T, class Op>
int go_bulk(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t k,
            const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  const size_t stage = (size_t)k * 32 * sizeof(T);
  // two stages (the block being stitched + the next block in flight): more
  // resident warps beat deeper per-warp prefetch (C5 f64: k=32 0.83 -> 0.71 ms,
  // k=128 1.20 -> 0.92 ms for R = 4/3 -> 2)
  int R = 2;
  static const char* rs = getenv("EXSUM_BULK_R");  // measurement override
  if (rs && atoi(rs) >= 2 && atoi(rs) <= 6) R = atoi(rs);
  const size_t smem = 128 + R * stage;
  if (smem > 200 * 1024) return -1;
  const int64_t strips = inner / 32;
  const int64_t lines = strips * outer;
  const int64_t nblocks = (n + k - 1) / k;
  // enough warps in flight: ~8 per SM, at least 2 blocks per segment
  const int64_t want = (int64_t)num_sms() * 8;
  int64_t nseg = (want + lines - 1) / lines;
  int64_t max_seg = nblocks / 2;
  if (max_seg < 1) max_seg = 1;
  if (nseg > max_seg) nseg = max_seg;
  if (nseg < 1) nseg = 1;
  const int64_t seg_len = k * ((nblocks + nseg - 1) / nseg);
  nseg = (n + seg_len - 1) / seg_len;
  const int64_t items = lines * nseg;
  int64_t grid = items;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (grid > cap) grid = cap;
  typedef typename AccOf<T>::type Acc;
  Acc* tpart = nullptr;
  if (ex && ex->kind == 2 && std::is_same<Op, OpAdd>::value && grid <= ex->cap) {
    tpart = (Acc*)ex->buf;
    ex->done = 1;
    ex->ppr = grid;
  }
  if (ex) ex->n_out_done = 1;
  if (tpart) {
    if (smem > 48 * 1024) ensure_smem((const void*)k_strided_bulk<T, Op, true>, smem);
    k_strided_bulk<T, Op, true><<<(unsigned)grid, 32, smem, s>>>(in, out, outer, n, inner, (int)k,
                                                                 seg_len, nseg, R, total, tpart);
  } else {
    if (smem > 48 * 1024) ensure_smem((const void*)k_strided_bulk<T, Op, false>, smem);
    k_strided_bulk<T, Op, false><<<(unsigned)grid, 32, smem, s>>>(in, out, outer, n, inner, (int)k,
                                                                  seg_len, nseg, R, total, nullptr);
  }
  return 1;
}

}  // namespace

// Eligible when strips of 32 columns tile `inner` and rows are 16-byte aligned.
int launch_strided_bulk(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                        int64_t inner, int64_t k, const void* total, cudaStream_t s, PassExtra* ex) {
  if (inner % 32 != 0 || ((uintptr_t)in % 16) != 0 || ((uintptr_t)out % 16) != 0) return -1;
  if (dtype == F32 && op == ADD)
    return go_bulk<float, OpAdd>((const float*)in, (float*)out, outer, n, inner, k, (const double*)total, s, ex);
  if (dtype == F64 && op == ADD)
    return go_bulk<double, OpAdd>((const double*)in, (double*)out, outer, n, inner, k, (const double*)total, s, ex);
  if (dtype == I64 && op == ADD)
    return go_bulk<i64, OpAdd>((const i64*)in, (i64*)out, outer, n, inner, k, (const i64*)total, s, ex);
  if (dtype == I64 && op == MAX)
    return go_bulk<i64, OpMax>((const i64*)in, (i64*)out, outer, n, inner, k, nullptr, s, ex);
  return -2;
}

}  // namespace exsum
