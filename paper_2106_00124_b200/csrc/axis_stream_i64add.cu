// axis_stream_i64add.cu -- instantiations of axis_stream.cuh for i64 / OpAdd.
#include <type_traits>

#include "axis_stream.cuh"

namespace exsum {

template <class T, class Op, int C, int K1, int EX>
int go_axis_stream_c(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t nout,
                     const typename AccOf<T>::type* total, cudaStream_t s, PassExtra* ex) {
  typedef typename AccOf<T>::type Acc;
  constexpr int VE = 16 / sizeof(T);
  constexpr int N2 = 32 * C;
  constexpr int NT = N2 / VE;
  constexpr int U = (16 / K1) * K1;
  const size_t smem = (size_t)2 * U * N2 * sizeof(T);
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm > 2048 / NT) per_sm = 2048 / NT;
  if (per_sm < 1) per_sm = 1;
  const int64_t strips = inner / N2;
  const int64_t lines = outer * strips;
  const int64_t nunits = (nout + U - 1) / U;
  int64_t nseg = pick_segments(lines, nunits, per_sm);
  const int64_t seg_len = U * ((nunits + nseg - 1) / nseg);
  nseg = (nout + seg_len - 1) / seg_len;
  const int64_t items = lines * nseg;
  int64_t grid = items;
  const int64_t cap = (int64_t)num_sms() * per_sm * 4;
  if (EX == 2 && cap > ex->cap) return -1;
  if (grid > cap) grid = cap;
  ensure_smem((const void*)k_axis_stream<T, Op, C, K1, EX>, smem);
  k_axis_stream<T, Op, C, K1, EX><<<(unsigned)grid, NT, smem, s>>>(
      in, out, outer, n, inner, nout, seg_len, nseg, total,
      EX == 1 ? (T*)ex->buf : nullptr, EX == 1 ? ex->row_len : N2,
      EX == 2 ? (Acc*)ex->buf : nullptr);
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
    if (inner % 1024 == 0 && (!ex || ex->kind != 1 || ex->row_len % 1024 == 0))
      return pick_axis_ex<T, Op, 32>(in, out, outer, n, inner, nout, k, total, s, ex);
  }
  if (inner % 512 == 0 && (!ex || ex->kind != 1 || ex->row_len % 512 == 0))
    return pick_axis_ex<T, Op, 16>(in, out, outer, n, inner, nout, k, total, s, ex);
  if (inner % 256 == 0 && (!ex || ex->kind != 1 || ex->row_len % 256 == 0))
    return pick_axis_ex<T, Op, 8>(in, out, outer, n, inner, nout, k, total, s, ex);
  return -1;
}

int launch_axis_stream_i64add(const void* in, void* out, int64_t outer, int64_t n, int64_t inner,
                             int64_t k, const void* total, cudaStream_t s, PassExtra* ex) {
  return go_axis_stream<i64, OpAdd>((const i64*)in, (i64*)out, outer, n, inner, k,
                                   (const typename AccOf<i64>::type*)total, s, ex);
}

}  // namespace exsum
