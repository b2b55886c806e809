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
//
// k_strided_tma (default where the tensor map applies): the same pipeline fed
// by 2-D TMA tensor tiles (cp.async.bulk.tensor, SASS UTMALDG) -- one
// elected lane issues a 32-column x 16-row box per chunk instead of 32 lanes
// issuing one 1-D copy per row -- and the ring is refilled progressively:
// as the prefix / combine loop of block b retires the 16 rows of chunk j of
// S_b, chunk j of block b + R is issued into them, so the next loads are in
// flight during the whole P loop and the following suffix loop (with
// whole-block refills they only overlapped the suffix loop).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>
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


// ---------------------------------------------------- 2-D TMA tensor tiles --
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kTmaRows = 16;  // rows per TMA box (chunk)

template <class T, class Op, bool TOT, bool EPI>
__global__ void __launch_bounds__(32)
k_strided_tma(const __grid_constant__ CUtensorMap map, T* __restrict__ out, int64_t outer, int64_t n,
              int64_t inner, int k, int64_t seg_len, int64_t nseg, int R,
              const typename AccOf<T>::type* __restrict__ total,
              typename AccOf<T>::type* __restrict__ tpart) {
  typedef typename AccOf<T>::type Acc;
  constexpr int B = kTmaRows;
  Acc tacc = Acc(0);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // R <= 15 barriers
  T* stg = reinterpret_cast<T*>(smem + 128);
  const int lane = threadIdx.x;
  const int nch = (k + B - 1) / B;                     // boxes per block
  const int64_t stage_elems = (int64_t)nch * B * 32;
  const uint32_t chunk_bytes = B * 32 * sizeof(T);
  T tot = T(0);
  if constexpr (EPI) tot = (T)(*total);
  const int64_t last_bs = (int64_t)k * ((n - 1) / k);
  const int64_t nb_total = (n + k - 1) / k;
  const int64_t strips = inner / 32;
  const int64_t items = strips * outer * nseg;
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    for (int i = 0; i < R; ++i) mbar_init(&bar[i], nch);  // one arrival per box
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t nload = 0, ncons = 0;  // running block load / consume counters -> stage, parity
  auto fin = [&](T v) -> T {
    if constexpr (EPI) return OpAdd::inverse<T>(tot, v);
    return v;
  };

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
    T* dst = out + o * n * inner + strip * 32 + lane;

    auto rows_of = [&](int64_t bi) -> int {
      const int64_t avail = n - bi * k;
      const int64_t want = bi == b_end ? k - 1 : k;  // the halo needs k-1 rows
      return (int)(avail < want ? avail : want);
    };
    // box j of block bi into its stage (rows past the array read as zeros and
    // are never used; a box may also cover rows of the next block -- unused)
    auto issue_box = [&](int64_t bi, uint32_t st, int j) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&bar[st], chunk_bytes);
        tma_load_3d(stg + st * stage_elems + (int64_t)j * B * 32, &map, (int)(strip * 32),
                    (int)(bi * k + j * B), (int)o, &bar[st]);
      }
    };
    auto issue = [&](int64_t bi) {
      fence_proxy_async_smem();
      __syncwarp();
      const uint32_t st = nload % R;
      for (int j = 0; j < nch; ++j) issue_box(bi, st, j);
      ++nload;
    };
    auto wait_idx = [&](uint32_t c) { mbar_wait(&bar[c % R], (c / R) & 1); };
    // in-block suffix (right nested), in place, in register batches of B rows
    // (all loads of a batch issue before its dependent chain)
    auto suffix = [&](T* blk, int rows) {
      if (rows % B == 0) {  // whole batches: no predicates
        T v;
        for (int hi = rows - 1; hi >= 0; hi -= B) {  // rows hi, hi-1, ..., hi-B+1
          T q[B];
#pragma unroll
          for (int i = 0; i < B; ++i) q[i] = blk[(hi - i) * 32 + lane];
          if (hi == rows - 1) {
            v = q[0];
            if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)v);
          } else {
            if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)q[0]);
            v = Op::apply(q[0], v);
            q[0] = v;
          }
#pragma unroll
          for (int i = 1; i < B; ++i) {
            if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)q[i]);
            v = Op::apply(q[i], v);
            q[i] = v;
          }
#pragma unroll
          for (int i = 0; i < B; ++i) blk[(hi - i) * 32 + lane] = q[i];
        }
        return;
      }
      T v = blk[(rows - 1) * 32 + lane];
      if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)v);
      for (int top = rows - 2; top >= 0; top -= B) {  // rows top, top-1, ..., top-B+1
        T q[B];
#pragma unroll
        for (int i = 0; i < B; ++i)
          if (top - i >= 0) q[i] = blk[(top - i) * 32 + lane];
#pragma unroll
        for (int i = 0; i < B; ++i)
          if (top - i >= 0) {
            if constexpr (TOT) tacc = OpAdd::apply<Acc>(tacc, (Acc)q[i]);
            v = Op::apply(q[i], v);
            q[i] = v;
          }
#pragma unroll
        for (int i = 0; i < B; ++i)
          if (top - i >= 0) blk[(top - i) * 32 + lane] = q[i];
      }
    };

    int64_t next_issue = b0;
    for (; next_issue < b0 + nblk && next_issue < b0 + R; ++next_issue) issue(next_issue);

    uint32_t cb = ncons;
    wait_idx(cb);
    T* cur = stg + (cb % R) * stage_elems;
    int len = rows_of(b0);
    suffix(cur, len);
    for (int64_t b = b0; b < b_end; ++b) {
      const int64_t bs = b * k;
      if (bs == last_bs) {  // last block: out = S
        for (int r = 0; r < len; ++r) st1(dst + (bs + r) * inner, fin(cur[r * 32 + lane]));
        break;
      }
      wait_idx(cb + 1);
      T* nxt = stg + ((cb + 1) % R) * stage_elems;
      const int nlen = rows_of(b + 1);
      // the block that refills cur's stage, box by box as its rows retire
      const bool refill = next_issue < b0 + nblk;
      const uint32_t rst = cb % R;
      // out[bs + r] = S[r] (+) P[r - 1], P[i] = nxt[0] (+) ... (+) nxt[i]
      // (r = 0: S only); rows of nxt past nlen leave P unchanged
      T P = nxt[lane];
      T* drow = dst + bs * inner;
      if (k % B == 0 && nlen == k) {
        // whole boxes, a whole next block: no predicates; row 0 is S alone
        T* dp = drow;
        for (int j = 0; j < nch; ++j) {
          const int r0 = j * B;
          T sv[B], pv[B];
#pragma unroll
          for (int i = 0; i < B; ++i) {
            sv[i] = cur[(r0 + i) * 32 + lane];
            pv[i] = nxt[(r0 + i - 1 + (r0 + i == 0)) * 32 + lane];  // row r-1 (row 0 unused)
          }
#pragma unroll
          for (int i = 0; i < B; ++i) {
            if (r0 + i >= 2) P = Op::apply(P, pv[i]);
            if (r0 + i >= 1) sv[i] = Op::apply(sv[i], P);
          }
#pragma unroll
          for (int i = 0; i < B; ++i) {
            st1(dp, fin(sv[i]));
            dp += inner;
          }
          if (refill) {
            fence_proxy_async_smem();
            __syncwarp();  // every lane has read these rows of S_b
            issue_box(next_issue, rst, j);
          }
        }
      } else
      for (int j = 0; j < nch; ++j) {
        const int r0 = j * B;
        T sv[B], pv[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
          const int r = r0 + i;
          if (r < k) {
            sv[i] = cur[r * 32 + lane];
            if (r >= 2 && r - 1 < nlen) pv[i] = nxt[(r - 1) * 32 + lane];
          }
        }
#pragma unroll
        for (int i = 0; i < B; ++i) {
          const int r = r0 + i;
          if (r < k && r >= 1) {
            if (r >= 2 && r - 1 < nlen) P = Op::apply(P, pv[i]);
            sv[i] = Op::apply(sv[i], P);
          }
        }
#pragma unroll
        for (int i = 0; i < B; ++i)
          if (r0 + i < k) st1(drow + (int64_t)(r0 + i) * inner, fin(sv[i]));
        if (refill) {
          fence_proxy_async_smem();
          __syncwarp();  // every lane has read these rows of S_b
          issue_box(next_issue, rst, j);
        }
      }
      if (refill) {
        ++nload;
        ++next_issue;
      }
      ++cb;
      if (b + 1 < b_end) {
        cur = nxt;
        len = nlen;
        suffix(cur, len);
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
#ifndef TMA_SMALL_SEG
#define TMA_SMALL_SEG 0
#endif
  // segments of >= 2 blocks bound the halo re-reads; an array too small to
  // fill the machine that way may take one-block segments
  int64_t max_seg = (TMA_SMALL_SEG && lines * (nblocks / 2) < want) ? nblocks : nblocks / 2;
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

PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
    cudaGetLastError();
  });
  return fn;
}

// The [outer, n, inner] array as a 3-D tensor (innermost first) with boxes of
// 32 columns x kTmaRows rows x 1; false when the map cannot describe it.
template <class T>
bool make_map(CUtensorMap* map, const T* in, int64_t outer, int64_t n, int64_t inner) {
  PFN_cuTensorMapEncodeTiled enc = encode_fn();
  if (!enc && getenv("EXSUM_VERBOSE")) fprintf(stderr, "exsum: no cuTensorMapEncodeTiled entry point\n");
  if (!enc || inner >= ((int64_t)1 << 31) || n >= ((int64_t)1 << 31) || outer >= ((int64_t)1 << 31))
    return false;
  const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : std::is_same<T, double>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                                                  : CU_TENSOR_MAP_DATA_TYPE_INT64;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)n, (cuuint64_t)outer};
  cuuint64_t strides[2] = {(cuuint64_t)(inner * sizeof(T)), (cuuint64_t)(n * inner * sizeof(T))};
  cuuint32_t box[3] = {32, kTmaRows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(map, dt, 3, const_cast<T*>(in), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("EXSUM_VERBOSE")) fprintf(stderr, "exsum: cuTensorMapEncodeTiled -> %d\n", (int)r);
  return r == CUDA_SUCCESS;
}

template <class T, class Op>
int go_tma(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t k,
           const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  static const char* off = getenv("EXSUM_TMA");  // 0: the 1-D bulk-copy kernel (measurement)
  if (off && off[0] == '0') return -1;
  if (k < kTmaRows || k > 4096) return -1;
  CUtensorMap map;
  if (!make_map(&map, in, outer, n, inner)) return -1;
  const int nch = (int)((k + kTmaRows - 1) / kTmaRows);
  const size_t stage = (size_t)nch * kTmaRows * 32 * sizeof(T);
  int R = 2;
  static const char* rs = getenv("EXSUM_BULK_R");  // measurement override
  if (rs && atoi(rs) >= 2 && atoi(rs) <= 6) R = atoi(rs);
  const size_t smem = 128 + R * stage;
  if (smem > 200 * 1024) return -1;
  const int64_t strips = inner / 32;
  const int64_t lines = strips * outer;
  const int64_t nblocks = (n + k - 1) / k;
  const int64_t want = (int64_t)num_sms() * 8;
  int64_t nseg = (want + lines - 1) / lines;
#ifndef TMA_SMALL_SEG
#define TMA_SMALL_SEG 0
#endif
  // segments of >= 2 blocks bound the halo re-reads; an array too small to
  // fill the machine that way may take one-block segments
  int64_t max_seg = (TMA_SMALL_SEG && lines * (nblocks / 2) < want) ? nblocks : nblocks / 2;
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
  auto go = [&](auto tot_c, auto epi_c) {
    constexpr bool TOT = decltype(tot_c)::value, EPI = decltype(epi_c)::value;
    ensure_smem((const void*)k_strided_tma<T, Op, TOT, EPI>, smem);
    k_strided_tma<T, Op, TOT, EPI><<<(unsigned)grid, 32, smem, s>>>(map, out, outer, n, inner, (int)k,
                                                                    seg_len, nseg, R, total, tpart);
  };
  using Y = std::true_type;
  using N = std::false_type;
  if constexpr (std::is_same<Op, OpAdd>::value) {
    if (tpart && total) go(Y(), Y());
    else if (tpart) go(Y(), N());
    else if (total) go(N(), Y());
    else go(N(), N());
  } else {
    go(N(), N());
  }
  return 1;
}

template <class T, class Op>
int go_large_k(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t k,
               const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  const int rc = go_tma<T, Op>(in, out, outer, n, inner, k, total, s, ex);
  if (rc >= 0) return rc;
  return go_bulk<T, Op>(in, out, outer, n, inner, k, total, s, ex);
}

}  // namespace

// Eligible when strips of 32 columns tile `inner` and rows are 16-byte aligned.
int launch_strided_bulk(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                        int64_t inner, int64_t k, const void* total, cudaStream_t s, PassExtra* ex) {
  if (inner % 32 != 0 || ((uintptr_t)in % 16) != 0 || ((uintptr_t)out % 16) != 0) return -1;
  if (dtype == F32 && op == ADD)
    return go_large_k<float, OpAdd>((const float*)in, (float*)out, outer, n, inner, k, (const double*)total, s, ex);
  if (dtype == F64 && op == ADD)
    return go_large_k<double, OpAdd>((const double*)in, (double*)out, outer, n, inner, k, (const double*)total, s, ex);
  if (dtype == I64 && op == ADD)
    return go_large_k<i64, OpAdd>((const i64*)in, (i64*)out, outer, n, inner, k, (const i64*)total, s, ex);
  if (dtype == I64 && op == MAX)
    return go_large_k<i64, OpMax>((const i64*)in, (i64*)out, outer, n, inner, k, nullptr, s, ex);
  return -2;
}

}  // namespace exsum
