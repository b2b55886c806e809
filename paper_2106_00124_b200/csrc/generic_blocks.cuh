// generic_blocks.cuh -- the any-k windowed pass (one thread per line block).
//
// Used for windows too large for the register-streaming kernels: strided
// axes with k > 32 (e.g. the (128,4,1) box of BASELINE config 5) and rows with
// k > 1024.  Same association as scan.py:61-102 (bit-exact).
#pragma once

#include "exsum_common.cuh"

namespace exsum {

// Any k: one thread per (column vector, block).  Sweep 1 writes the in-block
// suffixes S to `out`; sweep 2 re-reads them (the same thread just wrote
// them: L2 hits), runs the next block's prefix and finishes the stitch.
template <class T, class Op, int V>
__global__ void __launch_bounds__(256)
k_strided_blocks(const T* __restrict__ in, T* __restrict__ out, int64_t outer, int64_t n,
                 int64_t inner, int64_t k, const typename AccOf<T>::type* __restrict__ total) {
  typedef Vec<T, V> VT;
  const int64_t cv = inner / V;
  const int64_t nb = (n + k - 1) / k;
  const int64_t items = outer * cv * nb;
  const T tot = total ? (T)(*total) : T(0);
  const bool epi = total != nullptr;
  const int64_t last_bs = k * ((n - 1) / k);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < items;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t % cv;
    const int64_t rest = t / cv;
    const int64_t o = rest % outer;
    const int64_t b = rest / outer;
    const int64_t bs = b * k;
    const int64_t be = bs + k < n ? bs + k : n;
    const T* pin = in + o * n * inner + c * V;
    T* pout = out + o * n * inner + c * V;
    // sweep 1: in-block suffix (right nested), S -> out
    VT S = ld_stream<T, V>(pin + (be - 1) * inner);
    const bool last = bs == last_bs;
    if (last && epi) {
      VT w;
#pragma unroll
      for (int j = 0; j < V; ++j) w.v[j] = OpAdd::inverse<T>(tot, S.v[j]);
      st_stream<T, V>(pout + (be - 1) * inner, w);
    } else {
      *reinterpret_cast<VT*>(pout + (be - 1) * inner) = S;
    }
    for (int64_t x = be - 2; x >= bs; --x) {
      VT a = ld_stream<T, V>(pin + x * inner);
#pragma unroll
      for (int j = 0; j < V; ++j) S.v[j] = Op::apply(a.v[j], S.v[j]);
      VT w = S;
      if (epi && (last || x == bs)) {
#pragma unroll
        for (int j = 0; j < V; ++j) w.v[j] = OpAdd::inverse<T>(tot, w.v[j]);
      }
      *reinterpret_cast<VT*>(pout + x * inner) = w;
    }
    if (last) continue;
    // sweep 2: next block's left-nested prefix, stitched onto S
    const int64_t ns = be;
    const int64_t ne = ns + k < n ? ns + k : n;
    VT P = ld_stream<T, V>(pin + ns * inner);
    for (int64_t r = 1; r < k; ++r) {
      const int64_t p = ns + r - 1;  // P index min(x+k-1, n-1)
      if (p > ns && p < ne) {
        VT a = ld_stream<T, V>(pin + p * inner);
#pragma unroll
        for (int j = 0; j < V; ++j) P.v[j] = Op::apply(P.v[j], a.v[j]);
      }
      VT s = *reinterpret_cast<const VT*>(pout + (bs + r) * inner);
      VT w;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        T v = Op::apply(s.v[j], P.v[j]);
        w.v[j] = epi ? OpAdd::inverse<T>(tot, v) : v;
      }
      st_stream<T, V>(pout + (bs + r) * inner, w);
    }
  }
}

}  // namespace exsum
