// outer_pair.cu -- two consecutive strided passes in one pass over HBM.
//
// bdbs_included runs windowed_sum_axis (reference pkg/src/exsum/scan.py:61-102)
// along every axis in order (included.py:124-129).  For two consecutive
// non-contiguous axes a, a+1 of small extent (the dimension sweep's 28^5 and
// 16^6: 28 x 28 and 16 x 16) the pair of passes only mixes elements of one
// (a, a+1) plane per column of the remaining axes, so a CTA can take the whole
// NA x NB plane for a strip of S = 16 columns (64 / 128 bytes),
// run both passes in shared memory, and write the strip back once: 2 N s
// bytes for the two passes instead of 4 N s.
//
// B200 mapping:
//   * the strip's NA*NB rows of 64-128 bytes (consecutive CTAs take
//     consecutive strips, so the array streams) arrive as 16-byte cp.async
//     copies, the whole tile in flight; they leave as 16-byte streaming stores
//     with the BDBSC complement epilogue;
//   * shared layout [xa][xb][c] with c contiguous: a warp walks 32 lines that
//     differ in c (and xb), so both passes are bank-conflict-free unpadded;
//   * each line walk is the compile-time unrolled one of block_fused.cu
//     (bf_line_c: same association, bit-identical floats).
#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

namespace {

template <class T, class Op, int K, int N, class At>
__device__ __forceinline__ void op_line(At at) {
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

// strip width: 16 columns (64 bytes of float32, 128 of int64 / float64).
// Measured: float32 strips of 64 bytes beat 128 (C3d 0.044 -> 0.041 ms: a
// 28 x 28 x 16 tile is 50 KB, 4 CTAs per SM instead of 2), 8-byte strips of
// 64 bytes lost (0.059 -> 0.063 ms)
constexpr int OP_S = 16;

template <class T, class Op, int K, int NA, int NB>
__global__ void __launch_bounds__(1024)
k_outer_pair(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t inner,
             int pass_a, int pass_b, const typename AccOf<T>::type* __restrict__ total) {
  constexpr int S = OP_S;  // strip columns
  constexpr int VE = 16 / sizeof(T);
  constexpr int SV = S / VE;          // vectors per strip row
  constexpr int ROWS = NA * NB;
  typedef Vec<T, VE> VT;
  extern __shared__ __align__(16) unsigned char smem[];
  T* sm = reinterpret_cast<T*>(smem);
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t strips = inner / S;
  const int64_t tiles = outer * strips;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t o = tile / strips;
    const int64_t c0 = (tile - o * strips) * S;
    const T* src = in + o * ROWS * inner + c0;
    T* dst = out + o * ROWS * inner + c0;
    for (int q = tid; q < ROWS * SV; q += nt) {
      const int row = q / SV;
      const int v = q - row * SV;
      cp_async_n<16>(sm + row * S + v * VE, src + row * inner + v * VE);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (pass_a) {  // along xa: lines (xb, c), stride NB*S
      for (int L = tid; L < NB * S; L += nt) {
        T* p = sm + L;
        op_line<T, Op, K, NA>([&](int r) { return p + r * (NB * S); });
      }
      __syncthreads();
    }
    if (pass_b) {  // along xb: lines (xa, c), stride S
      for (int L = tid; L < NA * S; L += nt) {
        const int xa = L / S;
        T* p = sm + xa * NB * S + (L - xa * S);
        op_line<T, Op, K, NB>([&](int r) { return p + r * S; });
      }
      __syncthreads();
    }
    for (int q = tid; q < ROWS * SV; q += nt) {
      const int row = q / SV;
      const int v = q - row * SV;
      VT w = *reinterpret_cast<const VT*>(sm + row * S + v * VE);
      if (epi) {
#pragma unroll
        for (int j = 0; j < VE; ++j) w.v[j] = OpAdd::inverse<T>(tot, w.v[j]);
      }
      st_stream<T, VE>(dst + row * inner + v * VE, w);
    }
    __syncthreads();  // the next tile overwrites the stage
  }
}

template <class T, class Op, int K, int NA, int NB>
int go_outer(const T* in, T* out, int64_t outer, int64_t inner, int pass_a, int pass_b,
             const typename AccOf<T>::type* total, cudaStream_t s) {
  constexpr int S = OP_S;
  const size_t smem = (size_t)NA * NB * S * sizeof(T);
  // threads: the larger pass's lines in as few equal rounds as 1024 allow
  const int lines = (NA > NB ? NA : NB) * S;
  const int rounds = (lines + 1023) / 1024;
  int nt = ((lines + rounds - 1) / rounds + 31) / 32 * 32;
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm > 2048 / nt) per_sm = 2048 / nt;
  if (per_sm < 1) per_sm = 1;
  const int64_t tiles = outer * (inner / S);
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > tiles) grid = tiles;
  ensure_smem((const void*)k_outer_pair<T, Op, K, NA, NB>, smem);
  k_outer_pair<T, Op, K, NA, NB><<<(unsigned)grid, nt, smem, s>>>(in, out, outer, inner, pass_a,
                                                                  pass_b, total);
  return 1;
}

template <class T, class Op>
int go_outer_k(const T* in, T* out, int64_t outer, int64_t na, int64_t nb, int64_t inner,
               int64_t ka, int64_t kb, const typename AccOf<T>::type* total, cudaStream_t s) {
  const int64_t k = ka > 1 ? ka : kb;
  if ((ka > 1 && ka != k) || (kb > 1 && kb != k)) return 0;
  const int pa = ka > 1, pb = kb > 1;
  if (na != nb) return 0;
#define EXSUM_OP_N(NN)                                                                     \
  if (na == NN) {                                                                          \
    switch (k) {                                                                           \
      case 2: return go_outer<T, Op, 2, NN, NN>(in, out, outer, inner, pa, pb, total, s);  \
      case 4: return go_outer<T, Op, 4, NN, NN>(in, out, outer, inner, pa, pb, total, s);  \
      case 8:                                                                              \
        if constexpr (sizeof(T) == 4)                                                      \
          return go_outer<T, Op, 8, NN, NN>(in, out, outer, inner, pa, pb, total, s);      \
        return 0;                                                                          \
    }                                                                                      \
    return 0;                                                                              \
  }
  EXSUM_OP_N(16)
  EXSUM_OP_N(28)
#undef EXSUM_OP_N
  return 0;
}

}  // namespace

int outer_pair_ok(int dtype, int op, int64_t na, int64_t nb, int64_t inner, int64_t ka, int64_t kb) {
  if (getenv("EXSUM_OUTER_PAIR") && atoi(getenv("EXSUM_OUTER_PAIR")) == 0) return 0;
  if (!((dtype == F32 && op == ADD) || (dtype == F64 && op == ADD) || (dtype == I64 && op == ADD) ||
        (dtype == I64 && op == MAX)))
    return 0;
  const int64_t S = OP_S;
  if (na != nb || !(na == 16 || na == 28) || inner % S != 0) return 0;
  const int64_t k = ka > 1 ? ka : kb;
  if (ka <= 1 || kb <= 1 || ka != kb) return 0;  // two real passes with one window
  if (!(k == 2 || k == 4 || (k == 8 && dtype_size(dtype) == 4))) return 0;
  return 1;
}

int launch_outer_pair(int dtype, int op, const void* in, void* out, int64_t outer, int64_t na,
                      int64_t nb, int64_t inner, int64_t ka, int64_t kb, const void* total,
                      cudaStream_t s) {
  if (((uintptr_t)in % 16) || ((uintptr_t)out % 16)) return 0;
  if (dtype == F32 && op == ADD)
    return go_outer_k<float, OpAdd>((const float*)in, (float*)out, outer, na, nb, inner, ka, kb,
                                    (const double*)total, s);
  if (dtype == F64 && op == ADD)
    return go_outer_k<double, OpAdd>((const double*)in, (double*)out, outer, na, nb, inner, ka, kb,
                                     (const double*)total, s);
  if (dtype == I64 && op == ADD)
    return go_outer_k<i64, OpAdd>((const i64*)in, (i64*)out, outer, na, nb, inner, ka, kb,
                                  (const i64*)total, s);
  if (dtype == I64 && op == MAX)
    return go_outer_k<i64, OpMax>((const i64*)in, (i64*)out, outer, na, nb, inner, ka, kb, nullptr,
                                  s);
  return 0;
}

}  // namespace exsum
