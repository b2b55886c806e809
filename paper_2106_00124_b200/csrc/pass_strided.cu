// pass_strided.cu -- windowed pass along a non-contiguous axis (inner > 1).
//
// Restates windowed_sum_axis (reference pkg/src/exsum/scan.py:61-102) for a
// view [outer, n, inner]: every "column" (o, i) is an independent line of
// length n with element stride `inner`.
//
// B200 mapping: one thread owns V adjacent columns (a 4/8/16-byte vector) and
// walks its line block by block, so consecutive lanes touch consecutive
// columns and every row access of a warp is one coalesced 128-512 B run.  The
// thread keeps the in-block suffixes S of the current block and the raw values
// of the next block in registers (2*KMAX*V values): per block it issues KMAX
// independent vector loads (memory-level parallelism), computes the next
// block's running prefix P, emits out[x] = S[x] (+) P[min(x+k-1, n-1)], and
// turns the next block into suffixes in place.  Each element is read once and
// written once (2*N*s bytes, the compulsory traffic), except the k rows of
// halo a segment reads from its successor when a long axis is split across
// threads for occupancy.  The association is exactly the reference's, so the
// float results are bit-identical to it.
//
// k > 32 uses k_strided_blocks: one thread per (column-vector, block) and
// two sweeps; the suffix sweep's results round-trip through the output buffer
// (L2-resident at that distance) so no per-thread block storage is needed.
#include <stdlib.h>
#include <string.h>

#include "exsum_common.cuh"
#include "exsum_launch.h"
#include "generic_blocks.cuh"

namespace exsum {

static int strided_mode();

// EXTRA: 0 plain; 1 also folds every raw row segment of 32*V elements into
// rowpart (the box-complement reduction R over the last axis, finished by
// k_rowpart_final); 2 also folds all raw values into one partial per CTA
// (the BDBSC total, finished by k_total_final).  Both reuse loads the pass
// makes anyway, saving a full read of the array.
template <class T, class Op, int KMAX, int V, int EXTRA = 0>
__global__ void __launch_bounds__(256)
k_strided_reg(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n,
              int64_t inner, int k, int64_t seg_len, int64_t nseg,
              const typename AccOf<T>::type* __restrict__ total, T* __restrict__ rowpart = nullptr,
              int64_t row_len = 0, typename AccOf<T>::type* __restrict__ tpart = nullptr,
              int64_t n_out = -1) {
  typedef Vec<T, V> VT;
  typedef typename AccOf<T>::type Acc;
  // rows produced along the axis: [0, nout) (a shard's own planes when the
  // input carries a halo of the next shard's planes beyond them)
  const int64_t nout = n_out < 0 ? n : n_out;
  Acc tacc[V];
#pragma unroll
  for (int j = 0; j < V; ++j) tacc[j] = Op::template identity<Acc>();
  const int lane = threadIdx.x & 31;
  // EXTRA == 1: fold the KMAX rows of a freshly loaded block across the warp's
  // 32 lanes with a multi-value butterfly (KMAX-1 + 5-log2(KMAX) shuffles for
  // KMAX rows, instead of 5 per row); lanes whose low bits are zero end up
  // holding one row's sum each and store it to rowpart[part][row].
  auto extra_block = [&](const VT (&blk)[KMAX], int nrows, int64_t o, int64_t x0, int64_t c) {
    if constexpr (EXTRA == 1) {
      T sv[KMAX];
#pragma unroll
      for (int r = 0; r < KMAX; ++r) {
        T sum = blk[r].v[0];
#pragma unroll
        for (int j = 1; j < V; ++j) sum = Op::apply(sum, blk[r].v[j]);
        sv[r] = r < nrows ? sum : Op::template identity<T>();
      }
      int rowbase = 0;
#pragma unroll
      for (int cnt = KMAX, off = 16; cnt > 1; cnt >>= 1, off >>= 1) {
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
      constexpr int LOWB = 32 / KMAX;  // lanes still sharing a row
#pragma unroll
      for (int off = LOWB >> 1; off >= 1; off >>= 1)
        sv[0] = Op::apply(sv[0], __shfl_xor_sync(0xffffffffu, sv[0], off));
      if ((lane & (LOWB - 1)) == 0 && rowbase < nrows) {
        const int64_t c0 = c - lane;  // the warp's first column vector
        const int64_t e = (o * n + x0 + rowbase) * inner + c0 * V;
        rowpart[(e / row_len) * (row_len / (32 * V)) + (e % row_len) / (32 * V)] = sv[0];
      }
    } else if constexpr (EXTRA == 2) {
#pragma unroll
      for (int r = 0; r < KMAX; ++r)
        if (r < nrows) {
#pragma unroll
          for (int j = 0; j < V; ++j) tacc[j] = Op::apply(tacc[j], (Acc)blk[r].v[j]);
        }
    }
  };
  const int64_t cv = inner / V;  // column vectors per outer slab
  const int64_t items = outer * cv * nseg;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t last_bs = (int64_t)k * ((n - 1) / k);

  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < items;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t % cv;
    const int64_t rest = t / cv;
    const int64_t o = rest % outer;
    const int64_t seg = rest / outer;
    const int64_t xs = seg * seg_len;
    const int64_t xe = xs + seg_len < nout ? xs + seg_len : nout;
    const T* pin = in + o * n * inner + c * V;
    T* pout = out + o * nout * inner + c * V;

    VT cur[KMAX];
    int64_t bs = xs;
    int len = (int)(n - bs < k ? n - bs : k);
#pragma unroll
    for (int r = 0; r < KMAX; ++r)
      if (r < len) cur[r] = ld_stream<T, V>(pin + (bs + r) * inner);
    if constexpr (EXTRA != 0) {
      const int64_t inseg = xe - bs;
      extra_block(cur, (int)(len < inseg ? len : inseg), o, bs, c);
    }
    // in-block suffix, right nested: S[r] = a[r] (+) S[r+1]   (scan.py:75-79)
#pragma unroll
    for (int r = KMAX - 2; r >= 0; --r)
      if (r < len - 1) {
#pragma unroll
        for (int j = 0; j < V; ++j) cur[r].v[j] = Op::apply(cur[r].v[j], cur[r + 1].v[j]);
      }

    for (;;) {
      if (bs == last_bs) {  // last block: out = S   (scan.py:91-99 skips it)
#pragma unroll
        for (int r = 0; r < KMAX; ++r)
          if (r < len) {
            VT w = cur[r];
            if (epi) {
#pragma unroll
              for (int j = 0; j < V; ++j) w.v[j] = OpAdd::inverse<T>(tot, w.v[j]);
            }
            st_stream<T, V>(pout + (bs + r) * inner, w);
          }
        break;
      }
      const int64_t ns = bs + k;
      const bool more = ns < xe;  // next block belongs to this segment
      // rows of the next block that are needed: all (more) or k-1 (halo)
      const int64_t avail = n - ns;
      const int want = more ? k : k - 1;
      const int nlen = (int)(avail < want ? avail : want);
      VT nxt[KMAX];
#pragma unroll
      for (int r = 0; r < KMAX; ++r)
        if (r < nlen) nxt[r] = ld_stream<T, V>(pin + (ns + r) * inner);
      if constexpr (EXTRA != 0) {
        const int64_t inseg = xe - ns;  // rows of this block inside the segment
        extra_block(nxt, more ? (int)(nlen < inseg ? nlen : inseg) : 0, o, ns, c);
      }

      // stitch (scan.py:88-102): out[bs] = S[bs]; out[bs+r] = S (+) P[min(r-1, nlen-1)]
      {
        VT w = cur[0];
        if (epi) {
#pragma unroll
          for (int j = 0; j < V; ++j) w.v[j] = OpAdd::inverse<T>(tot, w.v[j]);
        }
        st_stream<T, V>(pout + bs * inner, w);
      }
      VT P = nxt[0];
#pragma unroll
      for (int r = 1; r < KMAX; ++r) {
        if (r < k) {
          const int jj = r - 1;
          if (jj >= 1 && jj < nlen) {
#pragma unroll
            for (int j = 0; j < V; ++j) P.v[j] = Op::apply(P.v[j], nxt[jj].v[j]);
          }
          VT w;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            T v = Op::apply(cur[r].v[j], P.v[j]);
            w.v[j] = epi ? OpAdd::inverse<T>(tot, v) : v;
          }
          st_stream<T, V>(pout + (bs + r) * inner, w);
        }
      }
      if (!more) break;
      bs = ns;
      len = nlen;
#pragma unroll
      for (int r = KMAX - 2; r >= 0; --r)
        if (r < len - 1) {
#pragma unroll
          for (int j = 0; j < V; ++j) nxt[r].v[j] = Op::apply(nxt[r].v[j], nxt[r + 1].v[j]);
        }
#pragma unroll
      for (int r = 0; r < KMAX; ++r) cur[r] = nxt[r];
    }
  }
  if constexpr (EXTRA == 2) {
    __shared__ Acc sh[8];
    Acc ta = tacc[0];
#pragma unroll
    for (int j = 1; j < V; ++j) ta = Op::apply(ta, tacc[j]);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) ta = Op::apply(ta, __shfl_xor_sync(0xffffffffu, ta, d));
    if (lane == 0) sh[threadIdx.x >> 5] = ta;
    __syncthreads();
    if (threadIdx.x == 0) {
      Acc t = sh[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = Op::apply(t, sh[w]);
      tpart[blockIdx.x] = t;
    }
  }
}


// One thread per (column vector, block) with the block's suffixes in
// registers; the next block's raw values stream through a running prefix.
// For register-heavy tiles (8-byte elements with k > 16) this keeps 64 data
// registers per thread instead of 128, and gives N/k-way parallelism.  The
// next-block rows a thread reads are the rows its neighbour warp (same CTA,
// next block) loads at the same time, so the re-read is served by L1/L2.
template <class T, class Op, int KMAX, int V>
__global__ void __launch_bounds__(256)
k_strided_block_reg(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n,
                    int64_t inner, int k, const typename AccOf<T>::type* __restrict__ total) {
  typedef Vec<T, V> VT;
  const int64_t cv = inner / V;
  const int64_t nb = (n + k - 1) / k;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t last_bs = (int64_t)k * ((n - 1) / k);
  // thread layout: 32 column vectors x 8 blocks per CTA
  const int64_t cgroups = (cv + 31) / 32;
  const int64_t bgroups = (nb + 7) / 8;
  const int64_t items = outer * cgroups * bgroups;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t cg = it % cgroups;
    const int64_t rest = it / cgroups;
    const int64_t o = rest % outer;
    const int64_t bg = rest / outer;
    const int64_t c = cg * 32 + (threadIdx.x & 31);
    const int64_t b = bg * 8 + (threadIdx.x >> 5);
    if (c >= cv || b >= nb) continue;
    const int64_t bs = b * k;
    const int len = (int)(n - bs < k ? n - bs : k);
    const T* pin = in + o * n * inner + c * V;
    T* pout = out + o * n * inner + c * V;
    VT S[KMAX];
#pragma unroll
    for (int r = 0; r < KMAX; ++r)
      if (r < len) S[r] = ld_stream<T, V>(pin + (bs + r) * inner);
#pragma unroll
    for (int r = KMAX - 2; r >= 0; --r)
      if (r < len - 1) {
#pragma unroll
        for (int j = 0; j < V; ++j) S[r].v[j] = Op::apply(S[r].v[j], S[r + 1].v[j]);
      }
    if (bs == last_bs) {
#pragma unroll
      for (int r = 0; r < KMAX; ++r)
        if (r < len) {
          VT w = S[r];
#pragma unroll
          for (int j = 0; j < V; ++j) w.v[j] = epi ? OpAdd::inverse<T>(tot, w.v[j]) : w.v[j];
          st_stream<T, V>(pout + (bs + r) * inner, w);
        }
      continue;
    }
    const int64_t ns = bs + k;
    const int nlen = (int)(n - ns < k - 1 ? n - ns : k - 1);
    VT nx[KMAX];
#pragma unroll
    for (int r = 0; r < KMAX - 1; ++r)
      if (r < nlen) nx[r] = *reinterpret_cast<const VT*>(pin + (ns + r) * inner);
    {
      VT w = S[0];
#pragma unroll
      for (int j = 0; j < V; ++j) w.v[j] = epi ? OpAdd::inverse<T>(tot, w.v[j]) : w.v[j];
      st_stream<T, V>(pout + bs * inner, w);
    }
    VT P = nx[0];
#pragma unroll
    for (int r = 1; r < KMAX; ++r) {
      if (r < k) {
        const int jj = r - 1;
        if (jj >= 1 && jj < nlen) {
#pragma unroll
          for (int j = 0; j < V; ++j) P.v[j] = Op::apply(P.v[j], nx[jj].v[j]);
        }
        VT w;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const T v = Op::apply(S[r].v[j], P.v[j]);
          w.v[j] = epi ? OpAdd::inverse<T>(tot, v) : v;
        }
        st_stream<T, V>(pout + (bs + r) * inner, w);
      }
    }
  }
}

namespace {

int g_num_sms = 0;

template <class T, class Op, int KMAX, int V>
int go_reg(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int k,
           const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  const int64_t nout = (ex && ex->n_out >= 0) ? ex->n_out : n;
  const int64_t lines = outer * (inner / V);
  // split the axis into k-aligned segments until ~2 waves of 256-thread
  // blocks are resident; keep segments >= 16 blocks so the halo stays small
  const int64_t want_threads = (int64_t)num_sms() * 1536;
  int64_t nseg = (want_threads + lines - 1) / lines;
  const int64_t nblocks = (nout + k - 1) / k;
  // halo cost is one block per segment (re-read, mostly from L2 since the
  // neighbouring segment streams it at the same time): split only as far as
  // occupancy needs, down to 4 blocks per segment (2 for L2-resident arrays,
  // where the kernel is latency bound)
  const bool small = outer * n * inner * (int64_t)sizeof(T) < ((int64_t)64 << 20);
  int64_t max_seg = nblocks / (small ? 2 : 4);
  if (max_seg < 1) max_seg = 1;
  if (nseg > max_seg) nseg = max_seg;
  if (nseg < 1) nseg = 1;
  const int64_t seg_len = (int64_t)k * ((nblocks + nseg - 1) / nseg);
  nseg = (nout + seg_len - 1) / seg_len;
  const int64_t items = lines * nseg;
  int64_t grid = (items + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 64;
  if (grid > cap) grid = cap;
  typedef typename AccOf<T>::type Acc;
  if (ex) ex->n_out_done = 1;
  if (ex && ex->kind == 1 && ex->row_len % (32 * V) == 0 && (inner / V) % 32 == 0) {
    k_strided_reg<T, Op, KMAX, V, 1><<<(unsigned)grid, 256, 0, s>>>(
        in, out, outer, n, inner, k, seg_len, nseg, total, (T*)ex->buf, ex->row_len, nullptr, nout);
    ex->done = 1;
    ex->ppr = ex->row_len / (32 * V);
    return 1;
  }
  if (ex && ex->kind == 2 && grid <= ex->cap) {
    k_strided_reg<T, Op, KMAX, V, 2><<<(unsigned)grid, 256, 0, s>>>(
        in, out, outer, n, inner, k, seg_len, nseg, total, nullptr, 0, (Acc*)ex->buf, nout);
    ex->done = 1;
    ex->ppr = grid;
    return 1;
  }
  k_strided_reg<T, Op, KMAX, V><<<(unsigned)grid, 256, 0, s>>>(in, out, outer, n, inner, k,
                                                               seg_len, nseg, total, nullptr, 0,
                                                               nullptr, nout);
  return 1;
}

template <class T, class Op, int V>
int go_v(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t k,
         const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  // register tile 2*KMAX vectors of V elements: keep KMAX*WORDS <= 64
  // (128 data registers per thread; beyond that ptxas spills)
  constexpr int WORDS = (int)(sizeof(T) * V / 4);
  if (k <= 2) return go_reg<T, Op, 2, V>(in, out, outer, n, inner, (int)k, total, s, ex);
  if (k <= 4) return go_reg<T, Op, 4, V>(in, out, outer, n, inner, (int)k, total, s, ex);
  if (k <= 8) return go_reg<T, Op, 8, V>(in, out, outer, n, inner, (int)k, total, s, ex);
  if constexpr (WORDS <= 4) {
    if (k <= 16) return go_reg<T, Op, 16, V>(in, out, outer, n, inner, (int)k, total, s, ex);
  }
  if constexpr (WORDS <= 2) {
    if (k <= 32) return go_reg<T, Op, 32, V>(in, out, outer, n, inner, (int)k, total, s, ex);
  }
  return -1;  // caller retries with a narrower vector
}

template <class T, class Op>
int go_strided(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t k,
               const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  const uintptr_t a = (uintptr_t)in | (uintptr_t)out;
  // EXSUM_VMAX caps the vector width (measurements); piggy-backed reductions
  // prefer 8-byte vectors for f32 (half the registers: 2 CTAs per SM)
  static int vmax = -1;
  if (vmax < 0) {
    const char* e = getenv("EXSUM_VMAX");
    vmax = e ? atoi(e) : 0;
  }
  static int vextra = -1;  // EXSUM_VEXTRA: vector cap for passes with piggy-backed reductions
  if (vextra < 0) {
    const char* e = getenv("EXSUM_VEXTRA");
    vextra = e ? atoi(e) : 2;
  }
  int vcap = vmax > 0 ? vmax : 16;
  if (vmax == 0 && ex && ex->kind != 0 && sizeof(T) == 4 && k > 8) vcap = vextra;
  const bool v16 = vcap >= (int)(16 / sizeof(T)) && inner % (16 / sizeof(T)) == 0 && a % 16 == 0;
  const bool v8 = vcap >= 2 && sizeof(T) == 4 && inner % 2 == 0 && a % 8 == 0;  // 8-byte (float2)
  if (strided_mode() == 4 || (k > 32 && strided_mode() != 1)) {
    // fall through to the per-block two-sweep kernel below
  } else if (strided_mode() == 3 || (k > 16 && k <= 32 && sizeof(T) == 8 && strided_mode() != 1)) {
    const int64_t cv = inner;
    const int64_t nb = (n + k - 1) / k;
    const int64_t items = outer * ((cv + 31) / 32) * ((nb + 7) / 8);
    int64_t grid = items;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (grid > cap) grid = cap;
    k_strided_block_reg<T, Op, 32, 1><<<(unsigned)grid, 256, 0, s>>>(in, out, outer, n, inner,
                                                                     (int)k, total);
    return 1;
  }
  if (k <= 32 && strided_mode() != 4) {
    int rc = -1;
    if (v16) rc = go_v<T, Op, 16 / sizeof(T)>(in, out, outer, n, inner, k, total, s, ex);
    if (rc < 0 && v8) rc = go_v<T, Op, 2>(in, out, outer, n, inner, k, total, s, ex);
    if (rc < 0) rc = go_v<T, Op, 1>(in, out, outer, n, inner, k, total, s, ex);
    if (rc >= 0) return rc;
  }
  const int64_t nb = (n + k - 1) / k;
  const int V = v16 ? (int)(16 / sizeof(T)) : 1;
  const int64_t items = outer * (inner / V) * nb;
  int64_t grid = (items + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 64;
  if (grid > cap) grid = cap;
  if (V == 4)
    k_strided_blocks<T, Op, (sizeof(T) == 4 ? 4 : 2)><<<(unsigned)grid, 256, 0, s>>>(in, out, outer, n, inner, k, total);
  else if (V == 2)
    k_strided_blocks<T, Op, 2><<<(unsigned)grid, 256, 0, s>>>(in, out, outer, n, inner, k, total);
  else
    k_strided_blocks<T, Op, 1><<<(unsigned)grid, 256, 0, s>>>(in, out, outer, n, inner, k, total);
  return 1;
}

}  // namespace

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms = v > 0 ? v : 148;
  }
  return g_num_sms;
}

size_t dtype_size(int dtype) { return dtype == F32 ? 4 : 8; }

int launch_rows_pass(int dtype, int op, const void* in, void* out, int64_t rows, int64_t n,
                     int64_t k, const void* total, cudaStream_t s);

int launch_strided_bulk(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                        int64_t inner, int64_t k, const void* total, cudaStream_t s,
                        PassExtra* ex);
int launch_axis_stream_f32(const void*, void*, int64_t, int64_t, int64_t, int64_t, const void*,
                           cudaStream_t, PassExtra*);
int launch_axis_stream_f64(const void*, void*, int64_t, int64_t, int64_t, int64_t, const void*,
                           cudaStream_t, PassExtra*);
int launch_axis_stream_i64add(const void*, void*, int64_t, int64_t, int64_t, int64_t, const void*,
                              cudaStream_t, PassExtra*);
int launch_axis_stream_i64max(const void*, void*, int64_t, int64_t, int64_t, int64_t, const void*,
                              cudaStream_t, PassExtra*);

// EXSUM_AXIS_STREAM=0|1|2 (measurements): never / every eligible pass except
// those folding row partials / every eligible pass (default: with the
// register butterfly the cp.async ring beats k_strided_reg there too, C4
// row-partials pass 1.54 -> 1.42 ms)
static int axis_stream_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("EXSUM_AXIS_STREAM");
    mode = e ? atoi(e) : 2;
  }
  return mode;
}

// EXSUM_STRIDED=auto|reg|bulk|blockreg|blocks picks the strided kernel (for
// measurements); auto: register streaming while the register tile fits,
// the bulk-copy pipeline beyond.
static int strided_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("EXSUM_STRIDED");
    mode = 0;
    if (e && !strcmp(e, "reg")) mode = 1;
    if (e && !strcmp(e, "bulk")) mode = 2;
    if (e && !strcmp(e, "blockreg")) mode = 3;
    if (e && !strcmp(e, "blocks")) mode = 4;
  }
  return mode;
}

int launch_pass(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                int64_t inner, int64_t k, const void* total, cudaStream_t s, PassExtra* ex) {
  if (ex) {
    ex->done = 0;
    ex->n_out_done = 0;
  }
  if (ex && ex->n_out >= 0 && ex->n_out != n) {
    // a shard pass producing fewer rows than it reads: register streaming only
    // (callers fall back to a full-length pass into a temporary otherwise)
    if (inner == 1 || k > 32 || (dtype != F32 && k > 16)) return 0;
  }
  if (inner == 1) return launch_rows_pass(dtype, op, in, out, outer, n, k, total, s);
  const int mode = strided_mode();
  const bool big = k > 32 || (dtype != F32 && k > 16);
  const int am = axis_stream_mode();
  if (am == 2 || (am == 1 && !(ex && ex->kind == 1))) {
    int rc = -1;
    if (dtype == F32 && op == ADD) rc = launch_axis_stream_f32(in, out, outer, n, inner, k, total, s, ex);
    else if (dtype == F64 && op == ADD) rc = launch_axis_stream_f64(in, out, outer, n, inner, k, total, s, ex);
    else if (dtype == I64 && op == ADD) rc = launch_axis_stream_i64add(in, out, outer, n, inner, k, total, s, ex);
    else if (dtype == I64 && op == MAX) rc = launch_axis_stream_i64max(in, out, outer, n, inner, k, total, s, ex);
    if (rc >= 0) return rc;
  }
  if (mode == 2 || (mode == 0 && big)) {
    const int rc = launch_strided_bulk(dtype, op, in, out, outer, n, inner, k, total, s,
                                       ex && ex->kind == 2 ? ex : nullptr);
    if (rc >= 0) return rc;
  }
  if (dtype == F32 && op == ADD)
    return go_strided<float, OpAdd>((const float*)in, (float*)out, outer, n, inner, k,
                                    (const double*)total, s, ex);
  if (dtype == F64 && op == ADD)
    return go_strided<double, OpAdd>((const double*)in, (double*)out, outer, n, inner, k,
                                     (const double*)total, s, ex);
  if (dtype == I64 && op == ADD)
    return go_strided<i64, OpAdd>((const i64*)in, (i64*)out, outer, n, inner, k,
                                  (const i64*)total, s, ex);
  if (dtype == I64 && op == MAX)
    return go_strided<i64, OpMax>((const i64*)in, (i64*)out, outer, n, inner, k, nullptr, s, ex);
  return -2;
}

}  // namespace exsum
