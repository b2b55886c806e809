// block_fused.cu -- the windowed passes of the trailing m axes in one pass
// over HBM, for arrays whose trailing block fits in shared memory.
//
// bdbs_included runs windowed_sum_axis (reference pkg/src/exsum/scan.py:61-102)
// along axes 0..d-1 in order (included.py:124-129).  When the last m axes of a
// C-order array form a small contiguous block -- the higher-dimensional
// configurations of the dimension sweep, 28^5, 16^6, 64^4 -- every pass along
// those axes stays inside one block, so a CTA can stage G whole blocks in
// shared memory, run the m passes there in axis order, and write the result
// once: 2 N s bytes for the m passes instead of 2 m N s.
//
// B200 mapping:
//   * stage in with element-sized cp.async copies (the whole tile in flight),
//     out with coalesced 16-byte streaming stores; shared memory holds the blocks with the last axis padded
//     to an odd row length, so the row pass (thread per row) and the strided
//     passes (thread per column, consecutive threads on consecutive columns)
//     are both free of bank conflicts;
//   * one thread walks one line of the axis with the window K known at compile
//     time: block b's raw values and the next block's raw values rotate through
//     registers, so each pass reads and writes every shared element once;
//   * the association is the reference's (in-block right-nested suffix,
//     left-nested prefix of the next block, one stitch combine; the last block
//     keeps its suffix), so float results stay bit-identical;
//   * tiles of G blocks keep ~32 KB of shared memory per CTA: several CTAs per
//     SM overlap one tile's staging with another's passes.
// The BDBSC complement epilogue (excluded.py:72-75) rides on the stores.
#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

// x / d for x < 2^32 / d (tile-local indices): one high multiply; magic 0
// stands for d == 1 (ceil(2^32 / 1) does not fit 32 bits)
__device__ __forceinline__ uint32_t bf_div(uint32_t x, uint32_t magic) {
  return magic ? __umulhi(x, magic) : x;
}

// In-place windowed pass over one line p[0], p[st], ..., p[(n-1) st]
// (scan.py:72-102 restated with register rotation).
template <class T, class Op, int K>
__device__ __forceinline__ void bf_line(T* p, int n, int st) {
  T cur[K];
  const int l0 = n < K ? n : K;
#pragma unroll
  for (int r = 0; r < K; ++r)
    if (r < l0) cur[r] = p[r * st];
#pragma unroll 2
  for (int bs = 0; bs < n; bs += K) {
    const int blen = n - bs < K ? n - bs : K;
#pragma unroll
    for (int r = K - 2; r >= 0; --r)
      if (r < blen - 1) cur[r] = Op::apply(cur[r], cur[r + 1]);
    T* q = p + bs * st;
    if (bs + K >= n) {  // last block: out = S
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (r < blen) q[r * st] = cur[r];
      break;
    }
    const int nlen = n - bs - K < K ? n - bs - K : K;
    T nxt[K];
#pragma unroll
    for (int r = 0; r < K; ++r)
      if (r < nlen) nxt[r] = q[(K + r) * st];
    q[0] = cur[0];
    T P = nxt[0];
#pragma unroll
    for (int r = 1; r < K; ++r) {
      const int jj = r - 1;
      if (jj >= 1 && jj < nlen) P = Op::apply(P, nxt[jj]);
      q[r * st] = Op::apply(cur[r], P);
    }
#pragma unroll
    for (int r = 0; r < K; ++r) cur[r] = nxt[r];
  }
}

// K: the window of every fused axis with a pass (k > 1); the dimension sweep's
// boxes are cubic, so one compile-time window covers them
template <class T, class Op, int K, bool VEC>
__global__ void __launch_bounds__(256, 2)
k_block_fused(const T* __restrict__ in, T* __restrict__ out, int64_t nblocks, BlockSpec bs,
              const typename AccOf<T>::type* __restrict__ total) {
  constexpr int VE = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem[];
  T* sm = reinterpret_cast<T*>(smem);
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const int nl = bs.n[bs.m - 1];  // row length (last axis)
  const int rowp = bs.rowp;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t ntiles = (nblocks + bs.G - 1) / bs.G;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * bs.G;
    const int g = (int)(nblocks - b0 < bs.G ? nblocks - b0 : bs.G);
    const int E = g * (int)bs.B;  // elements of this tile
    const T* src = in + b0 * bs.B;
    T* dst = out + b0 * bs.B;
    // ---- stage in: element e -> shared (e / nl) * rowp + e % nl, as
    // element-sized cp.async copies (LDGSTS): lanes on consecutive elements
    // (coalesced), the whole tile in flight at once with no registers held --
    // register-staged 16-byte loads waited a DRAM latency per batch (C3
    // int64 28^5: 0.115 -> 0.077 ms)
    for (int e = tid; e < E; e += nt) {
      const int row = (int)bf_div((uint32_t)e, bs.magic_nl);
      cp_async_n<sizeof(T)>(sm + row * rowp + (e - row * nl), src + e);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // ---- the passes, axes in order (included.py:127)
    for (int j = 0; j < bs.m; ++j) {
      if (bs.k[j] > 1) {
        const int n = bs.n[j];
        if (j == bs.m - 1) {
          const int rows = E / nl;
          for (int r = tid; r < rows; r += nt) bf_line<T, Op, K>(sm + r * rowp, n, 1);
        } else {
          // lines: (outer o, inner i); inner runs over the valid elements of
          // the later axes, i -> (i / nl) * rowp + i % nl in the padded layout
          const int inner = bs.inner[j];       // valid elements after axis j
          const int inner_p = inner / nl * rowp;  // padded stride of axis j
          const int lines = E / n;              // = outer * inner
          auto line_at = [&](int L) -> T* {
            const int o = (int)bf_div((uint32_t)L, bs.magic_inner[j]);
            const int i = L - o * inner;
            const int ir = (int)bf_div((uint32_t)i, bs.magic_nl);
            return sm + (o * n * inner_p + ir * rowp + (i - ir * nl));
          };
          for (int L = tid; L < lines; L += nt) bf_line<T, Op, K>(line_at(L), n, inner_p);
        }
        __syncthreads();
      }
    }
    // ---- stage out (+ BDBSC complement)
    if constexpr (VEC) {
      for (int e = tid * VE; e < E; e += nt * VE) {
        Vec<T, VE> v;
        int row = (int)bf_div((uint32_t)e, bs.magic_nl);
        int col = e - row * nl;
#pragma unroll
        for (int j = 0; j < VE; ++j) {
          const T w = sm[row * rowp + col];
          v.v[j] = epi ? OpAdd::inverse<T>(tot, w) : w;
          if (++col == nl) {
            col = 0;
            ++row;
          }
        }
        st_stream<T, VE>(dst + e, v);
      }
    } else {
      for (int e = tid; e < E; e += nt) {
        const int row = (int)bf_div((uint32_t)e, bs.magic_nl);
        const T w = sm[row * rowp + (e - row * nl)];
        st1(dst + e, epi ? OpAdd::inverse<T>(tot, w) : w);
      }
    }
    __syncthreads();  // the next tile overwrites the stage
  }
}

// ---- cubic trailing blocks (every fused axis of length NL, M of them): the
// same passes with the line length, the strides and the line -> shared-memory
// map known at compile time.  The line walk unrolls completely -- no bounds
// tests, shared addresses as immediates off one base, the next block's loads
// free to issue ahead of the current block's stores -- which the runtime-shape
// kernel above cannot do (C3d 28^5: 63 thread instructions per element there,
// issue-bound at 64% busy).  Same association, bit-identical results.
template <class T, class Op, int K, int N, class At>
__device__ __forceinline__ void bf_line_c(At at) {
  constexpr int NB = (N + K - 1) / K;
  T cur[K];
#pragma unroll
  for (int r = 0; r < K; ++r)
    if (r < N) cur[r] = *at(r);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int bs = b * K;
    const int blen = N - bs < K ? N - bs : K;
#pragma unroll
    for (int r = K - 2; r >= 0; --r)
      if (r < blen - 1) cur[r] = Op::apply(cur[r], cur[r + 1]);
    if (b == NB - 1) {  // last block: out = S
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (r < blen) *at(bs + r) = cur[r];
    } else {
      const int nlen = N - bs - K < K ? N - bs - K : K;
      T nxt[K];
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (r < nlen) nxt[r] = *at(bs + K + r);
      *at(bs) = cur[0];
      T P = nxt[0];
#pragma unroll
      for (int r = 1; r < K; ++r) {
        const int jj = r - 1;
        if (jj >= 1 && jj < nlen) P = Op::apply(P, nxt[jj]);
        *at(bs + r) = Op::apply(cur[r], P);
      }
#pragma unroll
      for (int r = 0; r < K; ++r) cur[r] = nxt[r];
    }
  }
}

__host__ __device__ constexpr int bf_pow(int b, int e) { return e <= 0 ? 1 : b * bf_pow(b, e - 1); }

// the same walk over a line held in registers (the row pass: a thread loads
// its row as 16-byte vectors, walks it, stores it back as vectors)
template <class T, class Op, int K, int N>
__device__ __forceinline__ void bf_line_r(T (&v)[N]) {
  constexpr int NB = (N + K - 1) / K;
  T cur[K];
#pragma unroll
  for (int r = 0; r < K; ++r)
    if (r < N) cur[r] = v[r];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int bs = b * K;
    const int blen = N - bs < K ? N - bs : K;
#pragma unroll
    for (int r = K - 2; r >= 0; --r)
      if (r < blen - 1) cur[r] = Op::apply(cur[r], cur[r + 1]);
    if (b == NB - 1) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (r < blen) v[bs + r] = cur[r];
    } else {
      const int nlen = N - bs - K < K ? N - bs - K : K;
      T nxt[K];
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (r < nlen) nxt[r] = v[bs + K + r];
      v[bs] = cur[0];
      T P = nxt[0];
#pragma unroll
      for (int r = 1; r < K; ++r) {
        const int jj = r - 1;
        if (jj >= 1 && jj < nlen) P = Op::apply(P, nxt[jj]);
        v[bs + r] = Op::apply(cur[r], P);
      }
#pragma unroll
      for (int r = 0; r < K; ++r) cur[r] = nxt[r];
    }
  }
}

// padded row length of the cubic stage: whole 16-byte vectors, an odd number
// of them -- a thread's row as LDS.128 / STS.128 hits 8 distinct 16-byte bank
// groups per quarter warp, and rows start 16-byte aligned so the stage fills
// with 16-byte cp.async copies (float32 rows of 28 need no padding at all)
__host__ __device__ constexpr int bf_rp(int nl, int ve) {
  return (((nl + ve - 1) / ve) % 2 == 0 ? (nl + ve - 1) / ve + 1 : (nl + ve - 1) / ve) * ve;
}

// rows of exactly 4 vectors (float32 rows of 16: the 16^6 sweep) are not
// padded but XOR-swizzled: vector q of row r sits at q ^ ((r >> 1) & 3).  The
// row pass (a quarter warp on 8 rows, one vector each) then hits 8 distinct
// bank groups, and a warp on 32 consecutive columns (two whole rows) stays
// conflict-free -- the padded 20-wide rows conflicted 2-way there.
// Planes (the NL rows of one index of the block's axis M-2) are padded to a
// stride PS = NL (mod 128 bytes): a warp on 32 consecutive lines of the axis
// M-2 pass (columns of consecutive planes) then lands on 32 consecutive
// bank words -- unpadded 28 x 28 planes (784 = 16 mod 32 words) put two
// planes' columns on the same banks.
template <class T, int NL>
struct BfLayout {
  static constexpr int VE = 16 / sizeof(T);
  static constexpr int W = 128 / sizeof(T);  // elements per 128-byte bank row
  static constexpr int V = NL / VE;
  static constexpr bool SWZ = V == 4;
  static constexpr int RP = SWZ ? NL : bf_rp(NL, VE);
  static constexpr int PLANE = NL * RP;
  static constexpr int PS = PLANE + ((NL - PLANE) % W + W) % W;
  __device__ static __forceinline__ int sw(int row) { return SWZ ? (row >> 1) & 3 : 0; }
  __device__ static __forceinline__ int row_at(int row) { return (row / NL) * PS + (row % NL) * RP; }
  // shared offset of vector q of row `row`
  __device__ static __forceinline__ int vec_at(int row, int q) { return row_at(row) + (q ^ sw(row)) * VE; }
};

// the pass along block axis J (0 = outermost of the M fused axes)
template <class T, class Op, int K, int NL, int M, int J>
__device__ __forceinline__ void bf_pass_c(T* sm, int lines, int tid, int nt) {
  constexpr int VE = 16 / sizeof(T);
  typedef BfLayout<T, NL> Lay;
  constexpr int RP = Lay::RP;
  if constexpr (J == M - 1) {
    typedef Vec<T, VE> VT;
    for (int r = tid; r < lines; r += nt) {
      T v[NL];
#pragma unroll
      for (int q = 0; q < NL / VE; ++q) {
        const VT t = *reinterpret_cast<const VT*>(sm + Lay::vec_at(r, q));
#pragma unroll
        for (int j = 0; j < VE; ++j) v[q * VE + j] = t.v[j];
      }
      bf_line_r<T, Op, K, NL>(v);
#pragma unroll
      for (int q = 0; q < NL / VE; ++q) {
        VT t;
#pragma unroll
        for (int j = 0; j < VE; ++j) t.v[j] = v[q * VE + j];
        *reinterpret_cast<VT*>(sm + Lay::vec_at(r, q)) = t;
      }
    }
  } else {
    constexpr int INNER = bf_pow(NL, M - 1 - J);  // valid elements after axis J
    constexpr int RSTEP = INNER / NL;             // rows per step along axis J
    // element stride of axis J: one row (J = M-2) or whole planes
    constexpr int INNER_P = RSTEP == 1 ? RP : (RSTEP / NL) * Lay::PS;
    for (int L = tid; L < lines; L += nt) {
      const int o = L / INNER;
      const int i = L - o * INNER;
      const int ir = i / NL;
      const int c = i - ir * NL;
      const int row0 = o * NL * RSTEP + ir;
      if constexpr (Lay::SWZ && RSTEP == 1) {
        // rows advance by one along the line and row0 is a multiple of NL:
        // the swizzle of row0 + r is (r >> 1) & 3, known at compile time
        T* bt[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) bt[t] = sm + Lay::row_at(row0) + ((c / VE) ^ t) * VE + c % VE;
        bf_line_c<T, Op, K, NL>([&](int r) { return bt[(r >> 1) & 3] + r * RP; });
      } else {
        // rows advance by multiples of 16 (or no swizzle): one column offset
        T* p = sm + Lay::row_at(row0) + ((c / VE) ^ Lay::sw(row0)) * VE + c % VE;
        bf_line_c<T, Op, K, NL>([&](int r) { return p + r * INNER_P; });
      }
    }
  }
}

template <class T, class Op, int K, int NL, int M>
__global__ void __launch_bounds__(512)
k_block_cubic(const T* __restrict__ in, T* __restrict__ out, int64_t nblocks, int G, int passes,
              const typename AccOf<T>::type* __restrict__ total) {
  constexpr int VE = 16 / sizeof(T);
  typedef BfLayout<T, NL> Lay;
  constexpr int B = bf_pow(NL, M);
  static_assert(NL % VE == 0, "rows of whole 16-byte vectors");
  static_assert(!Lay::SWZ || NL % 16 == 0, "the swizzle assumes row0 % 8 == 0 per line");
  typedef Vec<T, VE> VT;
  extern __shared__ __align__(16) unsigned char smem[];
  T* sm = reinterpret_cast<T*>(smem);
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t ntiles = (nblocks + G - 1) / G;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b0 = tile * G;
    const int g = (int)(nblocks - b0 < G ? nblocks - b0 : G);
    const int E = g * B;
    const T* src = in + b0 * B;
    T* dst = out + b0 * B;
    // stage in: 16-byte cp.async copies into the padded rows
    for (int e = tid * VE; e < E; e += nt * VE) {
      const int row = e / NL;
      cp_async_n<16>(sm + Lay::vec_at(row, (e - row * NL) / VE), src + e);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int lines = E / NL;
    // passes: bit j set = axis j of the block has a window (> 1)
    if (passes & 1) { bf_pass_c<T, Op, K, NL, M, 0>(sm, lines, tid, nt); __syncthreads(); }
    if (passes & 2) { bf_pass_c<T, Op, K, NL, M, 1>(sm, lines, tid, nt); __syncthreads(); }
    if constexpr (M > 2) {
      if (passes & 4) { bf_pass_c<T, Op, K, NL, M, 2 % M>(sm, lines, tid, nt); __syncthreads(); }
    }
    // stage out (+ BDBSC complement): 16-byte shared loads, streaming stores
    for (int e = tid * VE; e < E; e += nt * VE) {
      const int row = e / NL;
      VT v = *reinterpret_cast<const VT*>(sm + Lay::vec_at(row, (e - row * NL) / VE));
      if (epi) {
#pragma unroll
        for (int j = 0; j < VE; ++j) v.v[j] = OpAdd::inverse<T>(tot, v.v[j]);
      }
      st_stream<T, VE>(dst + e, v);
    }
    __syncthreads();
  }
}

static uint32_t bf_magic(uint32_t d) {
  // ceil(2^32 / d): exact quotients for x < 2^32 / d; 0 marks d == 1
  return d <= 1 ? 0u : (uint32_t)((((uint64_t)1 << 32) + d - 1) / d);
}

static int64_t bf_env(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoll(e) : dflt;
}

int block_fused_plan(int dtype, int d, const int64_t* ext, const int64_t* k, int first_axis,
                     BlockSpec* out) {
  if (bf_env("EXSUM_BLOCK_FUSE", 1) == 0) return 0;
  const int64_t es = (int64_t)dtype_size(dtype);
  const int64_t budget = bf_env("EXSUM_BF_KB", 96) * 1024;
  const int64_t tile_target = bf_env("EXSUM_BF_TILE_KB", 32) * 1024;
  const int64_t nl = ext[d - 1];
  const int64_t rowp = nl | 1;  // odd padded row length
  // the largest m (>= 2 axes, not before first_axis) whose padded block fits,
  // with at least two passes inside and every window a supported size
  for (int m = d - first_axis < BF_MAX ? d - first_axis : BF_MAX; m >= 2; --m) {
    int64_t B = 1;
    for (int a = d - m; a < d; ++a) B *= ext[a];
    const int64_t bytes = B / nl * rowp * es;
    if (bytes > budget) continue;
    int passes = 0;
    bool ok = true;
    int64_t kw = 0;
    for (int a = d - m; a < d; ++a) {
      if (k[a] > 1) {
        ++passes;
        if (kw == 0) kw = k[a];
        if (k[a] != kw || !(kw == 2 || kw == 4 || (kw == 8 && es == 4))) ok = false;
      }
    }
    if (!ok || passes < 2) return 0;  // a smaller m has no more passes than this one
    BlockSpec bs;
    bs.m = m;
    bs.B = B;
    bs.rowp = (int)rowp;
    int64_t G = tile_target / bytes;
    if (G < 1) G = 1;
    if (G * B > (1 << 20)) G = ((int64_t)1 << 20) / B;  // tile-local indices stay small
    if (G < 1) return 0;
    bs.G = (int)G;
    int64_t inner = B;
    for (int j = 0; j < m; ++j) {
      bs.n[j] = (int)ext[d - m + j];
      bs.k[j] = (int)k[d - m + j];
      inner /= ext[d - m + j];
      bs.inner[j] = (int)inner;
      bs.magic_inner[j] = bf_magic((uint32_t)(inner > 0 ? inner : 1));
    }
    bs.magic_nl = bf_magic((uint32_t)nl);
    bs.K = (int)kw;
    // threads: one per line of the pass with the fewest lines (every pass
    // walks its lines sequentially, so idle threads only add CTA size)
    int64_t nmax = 1;
    for (int a = d - m; a < d; ++a)
      if (k[a] > 1 && ext[a] > nmax) nmax = ext[a];
    int64_t nt = (G * B / nmax + 31) / 32 * 32;
    bs.threads = (int)(nt < 64 ? 64 : (nt > 256 ? 256 : nt));
    bs.smem = (size_t)G * (size_t)bytes;
    *out = bs;
    return 1;
  }
  return 0;
}

template <class T, class Op, int K, int NL, int M>
static int go_cubic(const T* in, T* out, int64_t N, const BlockSpec& bs,
                    const typename AccOf<T>::type* total, cudaStream_t s) {
  constexpr int VE = 16 / sizeof(T);
  if constexpr (NL % VE != 0) {
    return 0;
  } else {
    if (((uintptr_t)in % 16) || ((uintptr_t)out % 16)) return 0;  // the runtime-shape kernel
    const int64_t nblocks = N / bs.B;
    int passes = 0;
    for (int j = 0; j < M; ++j)
      if (bs.k[j] > 1) passes |= 1 << j;
    const size_t smem = (size_t)bs.G * (bs.B / NL / NL) * BfLayout<T, NL>::PS * sizeof(T);
    if (smem > 200 * 1024) return 0;
    // threads: the tile's lines in as few equal rounds as 512 threads allow
    const int64_t lines = (int64_t)bs.G * bs.B / NL;
    const int64_t rounds = (lines + 511) / 512;
    int nt = (int)(((lines + rounds - 1) / rounds + 31) / 32 * 32);
    if (nt < 64) nt = 64;
    int per_sm = (int)((228 * 1024) / (smem + 1024));
    if (per_sm > 2048 / nt) per_sm = 2048 / nt;
    if (per_sm > 32) per_sm = 32;
    if (per_sm < 1) per_sm = 1;
    const int64_t ntiles = (nblocks + bs.G - 1) / bs.G;
    int64_t grid = (int64_t)num_sms() * per_sm;
    if (grid > ntiles) grid = ntiles;
    ensure_smem((const void*)k_block_cubic<T, Op, K, NL, M>, smem);
    k_block_cubic<T, Op, K, NL, M><<<(unsigned)grid, nt, smem, s>>>(in, out, nblocks, bs.G, passes,
                                                                    total);
    return 1;
  }
}

template <class T, class Op, int K>
static int go_block(const T* in, T* out, int64_t N, const BlockSpec& bs,
                    const typename AccOf<T>::type* total, cudaStream_t s) {
  // cubic blocks of the dimension sweep's shapes: the compile-time kernel
  bool cubic = bf_env("EXSUM_BF_CUBIC", 1) != 0 && (bs.m == 2 || bs.m == 3);
  for (int j = 1; j < bs.m; ++j) cubic = cubic && bs.n[j] == bs.n[0];
  if (cubic) {
    const int nl = bs.n[0];
    int rc = 0;
    if (bs.m == 3 && nl == 16) rc = go_cubic<T, Op, K, 16, 3>(in, out, N, bs, total, s);
    if (bs.m == 3 && nl == 28) rc = go_cubic<T, Op, K, 28, 3>(in, out, N, bs, total, s);
    if (bs.m == 2 && nl == 28) rc = go_cubic<T, Op, K, 28, 2>(in, out, N, bs, total, s);
    if (bs.m == 2 && nl == 32) rc = go_cubic<T, Op, K, 32, 2>(in, out, N, bs, total, s);
    if (bs.m == 2 && nl == 64) rc = go_cubic<T, Op, K, 64, 2>(in, out, N, bs, total, s);
    if (rc) return rc;
  }
  const int64_t nblocks = N / bs.B;
  int per_sm = (int)((228 * 1024) / (bs.smem + 1024));
  if (per_sm > 2048 / bs.threads) per_sm = 2048 / bs.threads;
  if (per_sm > 32) per_sm = 32;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = (nblocks + bs.G - 1) / bs.G;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > ntiles) grid = ntiles;
  const bool vec = ((uintptr_t)in % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                   ((bs.B * (int64_t)sizeof(T)) % 16 == 0);
  if (vec) {
    ensure_smem((const void*)k_block_fused<T, Op, K, true>, bs.smem);
    k_block_fused<T, Op, K, true><<<(unsigned)grid, bs.threads, bs.smem, s>>>(in, out, nblocks, bs,
                                                                             total);
  } else {
    ensure_smem((const void*)k_block_fused<T, Op, K, false>, bs.smem);
    k_block_fused<T, Op, K, false><<<(unsigned)grid, bs.threads, bs.smem, s>>>(in, out, nblocks, bs,
                                                                              total);
  }
  return 1;
}

template <class T, class Op>
static int go_block_k(const T* in, T* out, int64_t N, const BlockSpec& bs,
                      const typename AccOf<T>::type* total, cudaStream_t s) {
  switch (bs.K) {
    case 2: return go_block<T, Op, 2>(in, out, N, bs, total, s);
    case 4: return go_block<T, Op, 4>(in, out, N, bs, total, s);
    // windows of 16 (and 8 for 8-byte lines) spill at two CTAs per SM; the
    // plan rejects them
    case 8:
      if constexpr (sizeof(T) == 4) return go_block<T, Op, 8>(in, out, N, bs, total, s);
      return -1;
  }
  return -1;
}

int launch_block_fused(int dtype, int op, const void* in, void* out, int64_t N, const BlockSpec& bs,
                       const void* total, cudaStream_t s) {
  if (dtype == F32 && op == ADD)
    return go_block_k<float, OpAdd>((const float*)in, (float*)out, N, bs, (const double*)total, s);
  if (dtype == F64 && op == ADD)
    return go_block_k<double, OpAdd>((const double*)in, (double*)out, N, bs, (const double*)total, s);
  if (dtype == I64 && op == ADD)
    return go_block_k<i64, OpAdd>((const i64*)in, (i64*)out, N, bs, (const i64*)total, s);
  if (dtype == I64 && op == MAX)
    return go_block_k<i64, OpMax>((const i64*)in, (i64*)out, N, bs, nullptr, s);
  return -2;
}

}  // namespace exsum
