// sat.cu -- summed-area-table routes ("sat", "satc") and the mod-add:<m>
// element maps.
//
// Reference (pkg/src/exsum):
//   sat_build        included.py:37-42   copy, then ops.accumulate along axes
//                                         0..d-1 (np.add.accumulate: a
//                                         sequential running sum per line)
//   _query_table     included.py:78-95   identity below, last plane repeated
//                                         above (pure copies)
//   sat_included     included.py:98-121  2^d corner terms in
//                                         itertools.product((False, True))
//                                         order: the all-high corner copied,
//                                         then combine_into (even number of low
//                                         picks) / subtract_into (odd)
//   sat_excluded     excluded.py:83-85   fold(A) (-) sat_included
//   ModAddOps        monoid.py:235-286   np.add / np.subtract then np.remainder
//
// B200 mapping.  The table build is d streaming scans (memory-bound, 2Ns
// each): the contiguous axis runs lane-per-line through a padded shared tile
// (coalesced 32x32 tiles, each lane scans its own line sequentially), the
// strided axes run thread-per-16-byte-column-vector with 8 rows of loads in
// flight.  Both keep numpy's sequential association, so float tables are
// bit-identical to the reference.  When an axis has too few lines to fill the
// GPU, the scan is segmented (local scans, a scan of segment totals, a carry
// pass); integers stay exact, floats then differ by reassociation.  The query
// is one gather kernel: every output reads its 2^d corners (L2-resident
// neighbours), folds them in the reference's order and applies the route's
// epilogue (complement with the total, mod-add reduction) before its single
// store -- the padded query table is never materialised.
#include <type_traits>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {

// ------------------------------------------------------------------ scans --

// Inclusive running sum along the contiguous axis of [rows, n], in segments
// of L (nseg per row; nseg == 1: whole rows).  Work item = (row, segment);
// 32 items per warp, one per lane, staged through a padded 32x33 tile.
template <class T, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
k_scan_rows(const T* in, T* out, int64_t rows, int64_t n, int64_t L,
            int64_t nseg) {
  constexpr int W = 32;
  constexpr int STRIDE = W + 1;
  __shared__ T smem[WARPS][32 * STRIDE];
  const int lane = threadIdx.x & 31;
  T* sm = smem[threadIdx.x >> 5];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t items = rows * nseg;
  const int64_t groups = (items + 31) / 32;
  for (int64_t g = warp; g < groups; g += nwarps) {
    const int64_t i0 = g * 32;
    const int ni = items - i0 >= 32 ? 32 : (int)(items - i0);
    int64_t mybase = 0, mylen = 0;
    if (lane < ni) {
      const int64_t it = i0 + lane;
      const int64_t row = it / nseg, seg = it - row * nseg;
      mybase = row * n + seg * L;
      mylen = n - seg * L < L ? n - seg * L : L;
    }
    int64_t maxlen = mylen;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const int64_t v = __shfl_xor_sync(0xffffffffu, maxlen, o);
      maxlen = v > maxlen ? v : maxlen;
    }
    T acc = T(0);
    for (int64_t xo = 0; xo < maxlen; xo += W) {
      for (int r = 0; r < ni; ++r) {
        const int64_t b = __shfl_sync(0xffffffffu, mybase, r);
        const int64_t l = __shfl_sync(0xffffffffu, mylen, r);
        if (xo + lane < l) sm[r * STRIDE + lane] = ld1(in + b + xo + lane);
      }
      __syncwarp();
      if (lane < ni) {
        const int w = mylen - xo < W ? (int)(mylen - xo) : W;
        for (int x = 0; x < w; ++x) {
          const T v = sm[lane * STRIDE + x];
          acc = (xo == 0 && x == 0) ? v : OpAdd::apply(acc, v);  // numpy: out[0] = a[0]
          sm[lane * STRIDE + x] = acc;
        }
      }
      __syncwarp();
      for (int r = 0; r < ni; ++r) {
        const int64_t b = __shfl_sync(0xffffffffu, mybase, r);
        const int64_t l = __shfl_sync(0xffffffffu, mylen, r);
        if (xo + lane < l) st1(out + b + xo + lane, sm[r * STRIDE + lane]);
      }
      __syncwarp();
    }
  }
}

// Inclusive running sum along the middle axis of [outer, n, inner]; a thread
// owns VE consecutive columns (one 16-byte vector when inner allows) of one
// segment and walks it with U rows of loads in flight.  In place is allowed.
template <class T, int VE, int U>
__global__ void __launch_bounds__(256)
k_scan_strided(const T* in, T* out, int64_t outer, int64_t n,
               int64_t inner, int64_t L, int64_t nseg) {
  typedef Vec<T, VE> VT;
  const int64_t cols = inner / VE;
  const int64_t items = outer * cols * nseg;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = it % cols;
    const int64_t rest = it / cols;
    const int64_t o = rest % outer;
    const int64_t seg = rest / outer;
    const int64_t xs = seg * L;
    const int64_t xe = xs + L < n ? xs + L : n;
    const T* src = in + (o * n + xs) * inner + c * VE;
    T* dst = out + (o * n + xs) * inner + c * VE;
    VT acc;
    for (int64_t x = 0; x < xe - xs; x += U) {
      const int cnt = xe - xs - x < U ? (int)(xe - xs - x) : U;
      VT buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < cnt) buf[u] = *reinterpret_cast<const VT*>(src + (x + u) * inner);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < cnt) {
          if (x == 0 && u == 0) {
            acc = buf[0];
          } else {
#pragma unroll
            for (int j = 0; j < VE; ++j) acc.v[j] = OpAdd::apply(acc.v[j], buf[u].v[j]);
          }
          *reinterpret_cast<VT*>(dst + (x + u) * inner) = acc;
        }
    }
  }
}

// Segmented scans, step 2: T[o, s, i] = out[o, (s+1) L - 1, i] for s < nseg-1.
template <class T>
__global__ void k_seg_gather(const T* __restrict__ out, T* __restrict__ tot, int64_t outer,
                             int64_t n, int64_t inner, int64_t L, int64_t nseg) {
  const int64_t cnt = outer * (nseg - 1) * inner;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % inner;
    const int64_t rest = e / inner;
    const int64_t s = rest % (nseg - 1);
    const int64_t o = rest / (nseg - 1);
    tot[e] = out[(o * n + (s + 1) * L - 1) * inner + i];
  }
}

// Segmented scans, step 4: out[o, x, i] = Tscan[o, x/L - 1, i] (+) out[o, x, i]
// for x >= L (Tscan: inclusive scan of the segment totals).
template <class T>
__global__ void k_carry_add(T* __restrict__ out, const T* __restrict__ tscan, int64_t outer,
                            int64_t n, int64_t inner, int64_t L, int64_t nseg) {
  const int64_t cnt = outer * (n - L) * inner;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % inner;
    const int64_t rest = e / inner;
    const int64_t x = L + rest % (n - L);
    const int64_t o = rest / (n - L);
    const int64_t s = x / L;
    T* p = out + (o * n + x) * inner + i;
    *p = OpAdd::apply(tscan[(o * (nseg - 1) + s - 1) * inner + i], *p);
  }
}

// ------------------------------------------------------------ mod-add maps --

// floor modulus (np.remainder for m > 0) via a 64x64 high multiply:
// q = umulhi(u, floor((2^64-1)/m)) undershoots u/m by at most 2.
__device__ __forceinline__ i64 floor_mod(i64 v, const FastMod& fm) {
  const unsigned long long u =
      v >= 0 ? (unsigned long long)v : (unsigned long long)(-(v + 1));
  const unsigned long long q = __umul64hi(u, fm.inv);
  unsigned long long r = u - q * fm.m;
  while (r >= fm.m) r -= fm.m;
  return v >= 0 ? (i64)r : (i64)(fm.m - 1 - r);
}

// mode 0: out = v mod m (canonical form / final reduction; in may equal out);
// mode 1: out = (T mod m) (-) v, then mod m (rsubtract_scalar, monoid.py:274-276,
//         T = the wrapping int64 sum of the raw input, monoid.py:284-286).
__global__ void k_mod_map(const i64* __restrict__ in, i64* __restrict__ out, int64_t N, int mode,
                          FastMod fm, const i64* __restrict__ total) {
  const i64 tm = mode == 1 ? floor_mod(*total, fm) : 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const i64 v = ld1(in + e);
    st1(out + e, floor_mod(mode == 1 ? OpAdd::inverse<i64>(tm, v) : v, fm));
  }
}

// out[x] = in[x] on the slice where x_j == n_j - 1 for every axis j with
// fixed bit set (the elements no combine of bdbs touched, which keep their
// raw values under mod-add).
__global__ void k_copy_slice(const i64* __restrict__ in, i64* __restrict__ out, SliceSpec sp,
                             int64_t count) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t, idx = 0, stride = 1;
    for (int j = sp.d - 1; j >= 0; --j) {
      int64_t xj;
      if (sp.fixed[j]) {
        xj = sp.ext[j] - 1;
      } else {
        xj = r % sp.ext[j];
        r /= sp.ext[j];
      }
      idx += xj * stride;
      stride *= sp.ext[j];
    }
    out[idx] = in[idx];
  }
}

// -------------------------------------------------------------- the query --

// out[x] = fold of the 2^d corner terms (included.py:98-121) followed by the
// route's epilogue:
//   QUERY_PLAIN         sat
//   QUERY_COMPLEMENT    satc: total (-) q           (excluded.py:72-75)
//   QUERY_MOD           mod-add sat: q mod m
//   QUERY_MOD_COMPLEMENT mod-add satc: ((total mod m) (-) q) mod m
// D > 0 unrolls the corner loops for that dimensionality; D == 0 is generic.
template <class T, int D>
__global__ void __launch_bounds__(256)
k_sat_query(const T* __restrict__ S, T* __restrict__ out, QShape q, int64_t N,
            const typename AccOf<T>::type* __restrict__ total, int mode, FastMod fm) {
  const int d = D > 0 ? D : q.d;
  T tot = T(0);
  if (mode == QUERY_COMPLEMENT) tot = (T)(*total);
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < N;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t offhi[D > 0 ? D : EXSUM_QMAX], offlo[D > 0 ? D : EXSUM_QMAX];
    unsigned lo_ok = 0;
    int64_t r = f, base_hi = 0;
#pragma unroll
    for (int j = (D > 0 ? D : EXSUM_QMAX) - 1; j >= 0; --j) {
      if (j >= d) continue;
      int64_t xj;
      if (q.ext[j] <= 0x7fffffff && r <= 0x7fffffff) {
        const unsigned rr = (unsigned)r, ee = (unsigned)q.ext[j];
        xj = rr % ee;
        r = rr / ee;
      } else {
        xj = r % q.ext[j];
        r /= q.ext[j];
      }
      const int64_t hi = xj + q.k[j] - 1 < q.ext[j] - 1 ? xj + q.k[j] - 1 : q.ext[j] - 1;
      offhi[j] = hi * q.str[j];
      offlo[j] = (xj - 1) * q.str[j] - offhi[j];  // delta when axis j picks its low corner
      base_hi += offhi[j];
      if (xj > 0) lo_ok |= 1u << j;
    }
    T acc = S[base_hi];
    const int64_t terms = (int64_t)1 << d;
    for (int64_t p = 1; p < terms; ++p) {
      int64_t idx = base_hi;
      unsigned need = 0;
      int par = 0;
#pragma unroll
      for (int j = 0; j < (D > 0 ? D : EXSUM_QMAX); ++j) {
        if (j >= d) break;
        if ((p >> (d - 1 - j)) & 1) {  // axis j takes its low corner x_j - 1
          idx += offlo[j];
          need |= 1u << j;
          par ^= 1;
        }
      }
      const T v = (need & ~lo_ok) ? T(0) : S[idx];  // identity plane below the table
      acc = par ? OpAdd::inverse<T>(acc, v) : OpAdd::apply(acc, v);
    }
    if (mode == QUERY_COMPLEMENT) {
      acc = OpAdd::inverse<T>(tot, acc);
    } else if constexpr (std::is_same<T, i64>::value) {  // mod-add runs on int64
      if (mode == QUERY_MOD) {
        acc = floor_mod(acc, fm);
      } else if (mode == QUERY_MOD_COMPLEMENT) {
        acc = floor_mod(OpAdd::inverse<T>(floor_mod((i64)(*total), fm), acc), fm);
      }
    }
    out[f] = acc;
  }
}

// ---------------------------------------------------------------- launchers --

namespace {

int64_t grid_for(int64_t work, int threads, int per_sm) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (g > cap) g = cap;
  return g < 1 ? 1 : g;
}

template <class T>
int go_scan(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t L, int64_t nseg,
            cudaStream_t s) {
  if (inner == 1) {
    constexpr int WARPS = 4;
    const int64_t groups = (outer * nseg + 31) / 32;
    k_scan_rows<T, WARPS><<<(unsigned)grid_for(groups * 32, WARPS * 32, 16), WARPS * 32, 0, s>>>(
        in, out, outer, n, L, nseg);
    return 1;
  }
  constexpr int VE = 16 / sizeof(T);
  const bool vec = inner % VE == 0 && ((uintptr_t)in % 16) == 0 && ((uintptr_t)out % 16) == 0;
  if (vec) {
    const int64_t work = outer * (inner / VE) * nseg;
    k_scan_strided<T, VE, 8><<<(unsigned)grid_for(work, 256, 8), 256, 0, s>>>(in, out, outer, n,
                                                                             inner, L, nseg);
  } else {
    const int64_t work = outer * inner * nseg;
    k_scan_strided<T, 1, 8><<<(unsigned)grid_for(work, 256, 8), 256, 0, s>>>(in, out, outer, n,
                                                                           inner, L, nseg);
  }
  return 1;
}

template <class T>
int go_query(const T* S, T* out, const QShape& q, int64_t N, const void* total, int mode,
             const FastMod& fm, cudaStream_t s) {
  typedef typename AccOf<T>::type Acc;
  const Acc* tot = (const Acc*)total;
  const unsigned g = (unsigned)grid_for(N, 256, 8);
  switch (q.d) {
    case 1: k_sat_query<T, 1><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
    case 2: k_sat_query<T, 2><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
    case 3: k_sat_query<T, 3><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
    case 4: k_sat_query<T, 4><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
    case 5: k_sat_query<T, 5><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
    case 6: k_sat_query<T, 6><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
    default: k_sat_query<T, 0><<<g, 256, 0, s>>>(S, out, q, N, tot, mode, fm); break;
  }
  return 1;
}

}  // namespace

int launch_scan(int dtype, const void* in, void* out, int64_t outer, int64_t n, int64_t inner,
                int64_t L, int64_t nseg, cudaStream_t s) {
  switch (dtype) {
    case 0: return go_scan((const float*)in, (float*)out, outer, n, inner, L, nseg, s);
    case 1: return go_scan((const double*)in, (double*)out, outer, n, inner, L, nseg, s);
    case 2: return go_scan((const i64*)in, (i64*)out, outer, n, inner, L, nseg, s);
  }
  return -1;
}

int launch_seg_carry(int dtype, void* out, void* tot, int64_t outer, int64_t n, int64_t inner,
                     int64_t L, int64_t nseg, int step, cudaStream_t s) {
  const int64_t work = step == 0 ? outer * (nseg - 1) * inner : outer * (n - L) * inner;
  const unsigned g = (unsigned)grid_for(work, 256, 8);
#define EXSUM_SEG(T)                                                                          \
  if (step == 0)                                                                              \
    k_seg_gather<T><<<g, 256, 0, s>>>((const T*)out, (T*)tot, outer, n, inner, L, nseg);      \
  else                                                                                        \
    k_carry_add<T><<<g, 256, 0, s>>>((T*)out, (const T*)tot, outer, n, inner, L, nseg);       \
  return 1;
  switch (dtype) {
    case 0: { EXSUM_SEG(float) }
    case 1: { EXSUM_SEG(double) }
    case 2: { EXSUM_SEG(i64) }
  }
#undef EXSUM_SEG
  return -1;
}

int launch_sat_query(int dtype, const void* S, void* out, const QShape& q, int64_t N,
                     const void* total, int mode, const FastMod& fm, cudaStream_t s) {
  switch (dtype) {
    case 0: return go_query((const float*)S, (float*)out, q, N, total, mode, fm, s);
    case 1: return go_query((const double*)S, (double*)out, q, N, total, mode, fm, s);
    case 2: return go_query((const i64*)S, (i64*)out, q, N, total, mode, fm, s);
  }
  return -1;
}

int launch_mod_map(const void* in, void* out, int64_t N, int mode, const FastMod& fm,
                   const void* total, cudaStream_t s) {
  k_mod_map<<<(unsigned)grid_for(N, 256, 8), 256, 0, s>>>(
      (const i64*)in, (i64*)out, N, mode, fm, (const i64*)total);
  return 1;
}

int launch_copy_slice(const void* in, void* out, const SliceSpec& sp, int64_t count,
                      cudaStream_t s) {
  k_copy_slice<<<(unsigned)grid_for(count, 256, 8), 256, 0, s>>>((const i64*)in, (i64*)out, sp,
                                                                  count);
  return 1;
}

}  // namespace exsum
