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
template <class T, class Op, int WARPS, int W>
__global__ void __launch_bounds__(WARPS * 32)
k_scan_rows(const T* in, T* out, int64_t rows, int64_t n, int64_t L, int64_t nseg, int rev) {
  // W elements of each of 32 lines per chunk: CPL = W / 32 per lane and line
  // (4-byte types take 64: 256-byte runs per line and fetch)
  constexpr int CPL = W / 32;
  constexpr int STRIDE = W + 1;
  __shared__ T smem[WARPS][32 * STRIDE];
  __shared__ int64_t sbase[WARPS][32], slen[WARPS][32];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  T* sm = smem[wid];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t items = rows * nseg;
  const int64_t groups = (items + 31) / 32;
  for (int64_t g = warp; g < groups; g += nwarps) {
    const int64_t i0 = g * 32;
    int64_t mybase = 0, mylen = 0;
    if (i0 + lane < items) {
      const int64_t it = i0 + lane;
      const int64_t row = it / nseg, seg = it - row * nseg;
      // line position p = seg*L + x lives at row*n + p (or n-1-p reversed)
      mybase = row * n + (rev ? n - 1 - seg * L : seg * L);
      mylen = n - seg * L < L ? n - seg * L : L;
    }
    const int64_t dir = rev ? -1 : 1;
    __syncwarp();
    sbase[wid][lane] = mybase;
    slen[wid][lane] = mylen;
    int64_t maxlen = mylen;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const int64_t v = __shfl_xor_sync(0xffffffffu, maxlen, o);
      maxlen = v > maxlen ? v : maxlen;
    }
    __syncwarp();
    T acc = T(0);
    // 32 * CPL independent loads per chunk; the next chunk's loads are issued
    // as soon as the current one is staged, so they overlap its scan and stores
    T v[32 * CPL];
#pragma unroll
    for (int r = 0; r < 32; ++r)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int64_t l = slen[wid][r];
        const int x = c * 32 + lane;
        v[r * CPL + c] = x < l ? ld1(in + sbase[wid][r] + dir * x) : T(0);
      }
    for (int64_t xo = 0; xo < maxlen; xo += W) {
#pragma unroll
      for (int r = 0; r < 32; ++r)
#pragma unroll
        for (int c = 0; c < CPL; ++c) sm[r * STRIDE + c * 32 + lane] = v[r * CPL + c];
      __syncwarp();
      if (xo + W < maxlen) {
#pragma unroll
        for (int r = 0; r < 32; ++r)
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const int64_t l = slen[wid][r];
            const int64_t xn = xo + W + c * 32 + lane;
            v[r * CPL + c] = xn < l ? ld1(in + sbase[wid][r] + dir * xn) : T(0);
          }
      }
      if (mylen > xo) {
        const int w = mylen - xo < W ? (int)(mylen - xo) : W;
        if (w == W) {
#pragma unroll
          for (int x = 0; x < W; ++x) {
            const T t = sm[lane * STRIDE + x];
            acc = (xo == 0 && x == 0) ? t : Op::apply(acc, t);  // numpy: out[0] = a[0]
            sm[lane * STRIDE + x] = acc;
          }
        } else {
          for (int x = 0; x < w; ++x) {
            const T t = sm[lane * STRIDE + x];
            acc = (xo == 0 && x == 0) ? t : Op::apply(acc, t);
            sm[lane * STRIDE + x] = acc;
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int64_t l = slen[wid][r];
          const int64_t x = xo + c * 32 + lane;
          if (x < l) st1(out + sbase[wid][r] + dir * x, sm[r * STRIDE + c * 32 + lane]);
        }
      __syncwarp();
    }
  }
}

// Inclusive running sum along the middle axis of [outer, n, inner]; a thread
// owns VE consecutive columns (one 16-byte vector when inner allows) of one
// segment and walks it with U rows of loads in flight.  In place is allowed.
template <class T, class Op, int VE, int U>
__global__ void __launch_bounds__(256)
k_scan_strided(const T* in, T* out, int64_t outer, int64_t n,
               int64_t inner, int64_t L, int64_t nseg, int rev) {
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
    // line position p lives at row p (or n-1-p reversed)
    const int64_t step = rev ? -inner : inner;
    const int64_t first = rev ? n - 1 - xs : xs;
    const T* src = in + (o * n + first) * inner + c * VE;
    T* dst = out + (o * n + first) * inner + c * VE;
    VT acc;
    for (int64_t x = 0; x < xe - xs; x += U) {
      const int cnt = xe - xs - x < U ? (int)(xe - xs - x) : U;
      VT buf[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < cnt) buf[u] = *reinterpret_cast<const VT*>(src + (x + u) * step);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (u < cnt) {
          if (x == 0 && u == 0) {
            acc = buf[0];
          } else {
#pragma unroll
            for (int j = 0; j < VE; ++j) acc.v[j] = Op::apply(acc.v[j], buf[u].v[j]);
          }
          *reinterpret_cast<VT*>(dst + (x + u) * step) = acc;
        }
    }
  }
}

// Segmented scans, step 2: T[o, s, i] = out[o, (s+1) L - 1, i] for s < nseg-1.
template <class T>
__global__ void k_seg_gather(const T* __restrict__ out, T* __restrict__ tot, int64_t outer,
                             int64_t n, int64_t inner, int64_t L, int64_t nseg, int rev) {
  const int64_t cnt = outer * (nseg - 1) * inner;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % inner;
    const int64_t rest = e / inner;
    const int64_t s = rest % (nseg - 1);
    const int64_t o = rest / (nseg - 1);
    const int64_t pos = (s + 1) * L - 1;
    tot[e] = out[(o * n + (rev ? n - 1 - pos : pos)) * inner + i];
  }
}

// Segmented scans, step 4: out[o, x, i] = Tscan[o, x/L - 1, i] (+) out[o, x, i]
// for x >= L (Tscan: inclusive scan of the segment totals).
template <class T, class Op>
__global__ void k_carry_add(T* __restrict__ out, const T* __restrict__ tscan, int64_t outer,
                            int64_t n, int64_t inner, int64_t L, int64_t nseg, int rev) {
  const int64_t cnt = outer * (n - L) * inner;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % inner;
    const int64_t rest = e / inner;
    const int64_t x = L + rest % (n - L);
    const int64_t o = rest / (n - L);
    const int64_t s = x / L;
    T* p = out + (o * n + (rev ? n - 1 - x : x)) * inner + i;
    *p = Op::apply(tscan[(o * (nseg - 1) + s - 1) * inner + i], *p);
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

// Row form of the query for d >= 2 (DH = d-1 leading axes, compile time).
// A group of G lanes (G = the last extent rounded up to a power of two, <= 32)
// owns one output row x' = (x_0..x_{d-2}); the 2^DH source rows of S for the
// leading corner patterns are fixed for the whole row, so the per-element
// work is two shifted loads (hi = min(x+k-1, n-1), lo = x-1) per source row
// in the reference's product order (last axis fastest).  Rows are visited
// with axis 0 in stride-k0 order (x0 = r + j*k0, j fastest): output planes
// x0 and x0+k0 share the S plane x0+k0-1, so each S plane is fetched from
// HBM about once and re-read from L2.
template <class T, int DH>
__global__ void __launch_bounds__(256)
k_sat_query_rows(const T* __restrict__ S, T* __restrict__ out, QShape q, int64_t rows, int G,
                 const typename AccOf<T>::type* __restrict__ total, int mode, FastMod fm) {
  constexpr int NP = 1 << DH;
  const int64_t n = q.ext[DH];
  const int64_t kl = q.k[DH];
  const int lane = threadIdx.x & 31;
  const int slot = lane / G, sub = lane % G, slots = 32 / G;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n0 = q.ext[0], k0 = q.k[0];
  const int64_t per0 = rows / n0;  // rows per axis-0 plane
  T tot = T(0);
  if (mode == QUERY_COMPLEMENT) tot = (T)(*total);
  i64 tmod = 0;
  if constexpr (std::is_same<T, i64>::value) {
    if (mode == QUERY_MOD_COMPLEMENT) tmod = floor_mod((i64)(*total), fm);
  }
  for (int64_t rb = gwarp * slots; rb < rows; rb += nwarps * slots) {
    const int64_t ri = rb + slot;
    if (ri >= rows) continue;
    // permuted axis-0 order: plane index p -> x0 = (p % m) * k0 + p / m
    const int64_t p = ri / per0, rest = ri - p * per0;
    const int64_t m = (n0 + k0 - 1) / k0;
    const int64_t r0 = p / m, j0 = p - r0 * m;
    int64_t x0 = j0 * k0 + r0;
    int64_t hi_off[DH], lo_off[DH];
    unsigned lo_ok = 0;
    // the permutation is a bijection only when n0 % k0 == 0; otherwise fall
    // back to the identity order
    if (n0 % k0 != 0) x0 = p;
    {
      int64_t r = rest;
#pragma unroll
      for (int j = DH - 1; j >= 0; --j) {
        int64_t xj;
        if (j == 0) {
          xj = x0;
        } else {
          xj = r % q.ext[j];
          r /= q.ext[j];
        }
        const int64_t hi = xj + q.k[j] - 1 < q.ext[j] - 1 ? xj + q.k[j] - 1 : q.ext[j] - 1;
        hi_off[j] = hi * q.str[j];
        lo_off[j] = (xj - 1) * q.str[j];
        if (xj > 0) lo_ok |= 1u << j;
      }
    }
    int64_t obase = 0;
    {
      int64_t r = rest;
#pragma unroll
      for (int j = DH - 1; j >= 1; --j) {
        obase += (r % q.ext[j]) * q.str[j];
        r /= q.ext[j];
      }
      obase += x0 * q.str[0];
    }
    // the 2^DH source rows of this output row and which of them exist
    const T* src[NP];
    unsigned vmask = 0;
    int par_mask = 0;
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      int64_t base = 0;
      unsigned need = 0;
      int par = 0;
#pragma unroll
      for (int j = 0; j < DH; ++j) {
        if ((pp >> (DH - 1 - j)) & 1) {
          base += lo_off[j];
          need |= 1u << j;
          par ^= 1;
        } else {
          base += hi_off[j];
        }
      }
      src[pp] = S + ((need & ~lo_ok) == 0 ? base : 0);  // invalid: any readable row
      if ((need & ~lo_ok) == 0) vmask |= 1u << pp;
      par_mask |= par << pp;
    }
    T* dst = out + obase;
    const int nn = (int)n, kk = (int)kl;
    // one output element: unconditional loads (identity terms come from a
    // select, so signed zeros follow the reference's arithmetic exactly)
    auto element = [&](int x) -> T {
      const int hi = x + kk - 1 < nn - 1 ? x + kk - 1 : nn - 1;
      const int lo = x > 0 ? x - 1 : 0;
      T acc = T(0);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const bool valid = (vmask >> pp) & 1;
        // sign of the term: the parity of its low picks, a compile-time
        // constant of the unrolled pattern index (no per-element select)
        const bool par = __popc((unsigned)pp) & 1;
        const T h = __ldg(src[pp] + hi);
        const T l = __ldg(src[pp] + lo);
        const T vh = valid ? h : T(0);
        const T vl = (valid && x > 0) ? l : T(0);
        if (pp == 0) {
          acc = vh;  // the all-high corner is copied (included.py:116-117)
        } else {
          acc = par ? OpAdd::inverse<T>(acc, vh) : OpAdd::apply(acc, vh);
        }
        acc = par ? OpAdd::apply(acc, vl) : OpAdd::inverse<T>(acc, vl);
      }
      if (mode == QUERY_COMPLEMENT) {
        acc = OpAdd::inverse<T>(tot, acc);
      } else if constexpr (std::is_same<T, i64>::value) {
        if (mode == QUERY_MOD) {
          acc = floor_mod(acc, fm);
        } else if (mode == QUERY_MOD_COMPLEMENT) {
          acc = floor_mod(OpAdd::inverse<T>(tmod, acc), fm);
        }
      }
      return acc;
    };
    constexpr int XU = 4;  // x values per thread per step: XU * 2^(DH+1) loads in flight
    int xb = sub;
    for (; xb + (XU - 1) * G < nn; xb += XU * G) {
      T r[XU];
#pragma unroll
      for (int u = 0; u < XU; ++u) r[u] = element(xb + u * G);
#pragma unroll
      for (int u = 0; u < XU; ++u) st1(dst + xb + u * G, r[u]);
    }
    for (; xb < nn; xb += G) st1(dst + xb, element(xb));
  }
}

// Chained form of the staged query (d >= 2, long rows).  The last leading
// axis c = d-2 is walked in steps of k_c: for output rows x_c = r + j k_c the
// high corner of step j (row min(x_c + k_c - 1, n_c - 1)) is exactly the low
// corner (row x_c' - 1) of step j+1, so every step stages only the 2^(d-2)
// new high rows (one per pattern of the other leading axes) and reuses the
// previous step's rows from shared memory -- half the L2->SM traffic of a
// row-at-a-time form.  A 4-slot cp.async ring keeps two steps of prefetch in
// flight (Little's law: ~64 KB per SM at HBM latency).  A work item (chain) is (the other leading coordinates, r); chains
// are ordered so that CTAs running together share S planes in L2.
template <class T, int DH, int NT, int kChainThreads>
__global__ void __launch_bounds__(kChainThreads)
k_sat_query_chain(const T* __restrict__ S, T* __restrict__ out, QShape q, int64_t chains,
                  const typename AccOf<T>::type* __restrict__ total, int mode, FastMod fm) {
  constexpr int NQ = 1 << (DH - 1);  // patterns of the other leading axes
  constexpr int C = DH - 1;          // chain axis
  constexpr int VE = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);
  // NT > 0: the row length at compile time, so the per-pattern row offsets
  // below are immediates of the shared loads (no per-load address math)
  const int n = NT > 0 ? NT : (int)q.ext[DH];
  const int kl = (int)q.k[DH];
  const int pitch = n + VE;
  const int slot_elems = NQ * pitch;
  const int tid = threadIdx.x;
  const int64_t nc = q.ext[C], kc = q.k[C];
  const int64_t strc = q.str[C];
  T tot = T(0);
  if (mode == QUERY_COMPLEMENT) tot = (T)(*total);
  i64 tmod = 0;
  if constexpr (std::is_same<T, i64>::value) {
    if (mode == QUERY_MOD_COMPLEMENT) tmod = floor_mod((i64)(*total), fm);
  }
  for (int i = tid; i < 4 * NQ * VE; i += kChainThreads) buf[(i / VE) * pitch + (i % VE)] = T(0);
  __syncthreads();

  for (int64_t ch = blockIdx.x; ch < chains; ch += gridDim.x) {
    // chain -> (r, coordinates of axes 0..C-1); axis 0 in stride-k0 order
    const int64_t r = ch % kc;
    int64_t rest = ch / kc;
    int64_t xs[DH > 1 ? DH - 1 : 1];
    int64_t obase_lead = 0;
    {
#pragma unroll
      for (int j = C - 1; j >= 0; --j) {
        xs[j] = rest % q.ext[j];
        rest /= q.ext[j];
      }
      if (C >= 1 && q.ext[0] % q.k[0] == 0) {  // permute axis 0: x0 = (p % m) k0 + p / m
        const int64_t p = xs[0], m = q.ext[0] / q.k[0];
        xs[0] = (p % m) * q.k[0] + p / m;
      }
#pragma unroll
      for (int j = 0; j < C; ++j) obase_lead += xs[j] * q.str[j];
    }
    // per pattern q of axes 0..C-1: row offset (without the chain axis), validity, parity
    int64_t qoff[NQ];
    unsigned qvalid = 0;
    int qpar = 0;
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
      int64_t base = 0;
      bool ok = true;
      int par = 0;
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const bool lo = (qq >> (C - 1 - j)) & 1;
        const int64_t xj = xs[j];
        if (lo) {
          base += (xj - 1) * q.str[j];
          ok = ok && xj > 0;
          par ^= 1;
        } else {
          const int64_t hi = xj + q.k[j] - 1 < q.ext[j] - 1 ? xj + q.k[j] - 1 : q.ext[j] - 1;
          base += hi * q.str[j];
        }
      }
      qoff[qq] = base;
      if (ok) qvalid |= 1u << qq;
      qpar |= par << qq;
    }
    // stage the 2^(d-2) rows at chain-axis row cr (cr < 0: identity rows)
    auto stage = [&](int slot, int64_t cr) {
      T* b = buf + (size_t)slot * slot_elems + VE;
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        T* row = b + qq * pitch;
        if (((qvalid >> qq) & 1) && cr >= 0) {
          const T* g = S + qoff[qq] + cr * strc;
          for (int c = tid * VE; c < n; c += kChainThreads * VE) cp_async16(row + c, g + c);
        } else {
          for (int c = tid; c < n; c += kChainThreads) row[c] = T(0);
        }
      }
      cp_async_commit();
    };
    const int64_t steps = (nc - r + kc - 1) / kc;
    auto hi_row = [&](int64_t j) {
      const int64_t xc = r + j * kc;
      return xc + kc - 1 < nc - 1 ? xc + kc - 1 : nc - 1;
    };
    // ring of RING slots: step j reads slots j % RING (low) and (j+1) % RING
    // (high); the high rows of steps j+1 .. j+DEPTH are in flight
    constexpr int RING = 4, DEPTH = RING - 2;
    stage(0, r - 1);      // low rows of step 0
    stage(1, hi_row(0));  // high rows of step 0
#pragma unroll
    for (int d = 1; d <= DEPTH; ++d) {
      if (d < steps) stage(d + 1, hi_row(d));
      else cp_async_commit();  // empty group keeps the wait counts uniform
    }
    for (int64_t j = 0; j < steps; ++j) {
      const int lo_slot = (int)(j % RING), hi_slot = (int)((j + 1) % RING);
      cp_async_wait<DEPTH>();  // groups up to step j's high rows have landed
      __syncthreads();
      const int64_t xc = r + j * kc;
      const T* lob = buf + (size_t)lo_slot * slot_elems;
      const T* hib = buf + (size_t)hi_slot * slot_elems;
      T* dst = out + obase_lead + xc * strc;
      const int xmain = n - kl + 1;  // x < xmain: the high corner x + kl - 1 is in the row
      // compile-time row length: fully unrolled, so every x's shared and
      // global addresses are immediate offsets of this step's bases
#pragma unroll (NT > 0 ? (NT + kChainThreads - 1) / kChainThreads : 1)
      for (int x = tid; x < n; x += kChainThreads) {
        const int hi = VE + (x < xmain ? x + kl - 1 : n - 1);
        const int lo = VE - 1 + x;  // x - 1; the zero pad for x = 0
        // four base addresses; every pattern's row is a constant offset from one
        const T* lh = lob + hi;
        const T* ll = lob + lo;
        const T* hh = hib + hi;
        const T* hl = hib + lo;
        T acc = T(0);
#pragma unroll
        for (int pp = 0; pp < 2 * NQ; ++pp) {
          const int qq = pp >> 1;
          const bool clo = pp & 1;  // chain axis takes its low corner
          const bool par = ((__popc((unsigned)qq) + (int)clo) & 1) != 0;  // compile-time
          const T vh = (clo ? lh : hh)[qq * pitch];
          const T vl = (clo ? ll : hl)[qq * pitch];
          if (pp == 0) {
            acc = vh;  // the all-high corner is copied (included.py:116-117)
          } else {
            acc = par ? OpAdd::inverse<T>(acc, vh) : OpAdd::apply(acc, vh);
          }
          acc = par ? OpAdd::apply(acc, vl) : OpAdd::inverse<T>(acc, vl);
        }
        if (mode == QUERY_COMPLEMENT) {
          acc = OpAdd::inverse<T>(tot, acc);
        } else if constexpr (std::is_same<T, i64>::value) {
          if (mode == QUERY_MOD) {
            acc = floor_mod(acc, fm);
          } else if (mode == QUERY_MOD_COMPLEMENT) {
            acc = floor_mod(OpAdd::inverse<T>(tmod, acc), fm);
          }
        }
        st1(dst + x, acc);
      }
      __syncthreads();  // step j's low slot is refilled next, with step j+DEPTH+1's rows
      if (j + DEPTH + 1 < steps) stage((int)((j + DEPTH + 2) % RING), hi_row(j + DEPTH + 1));
      else cp_async_commit();
    }
    cp_async_wait<0>();
    __syncthreads();
  }
}

// ------------------------------------------------------------- corners --

// One corner pattern's contribution (excluded.py:218-234): along axis a the
// scanned copy is read at T-1 clamped to n-1 (prefix letter; nothing when
// T-1 < 0) or at T (suffix letter; nothing when T >= n), T = x (near face)
// or x + k (far face).  first: out starts from the identity (Tensor.filled).
template <class T, class Op>
__global__ void k_corner_apply(const T* __restrict__ sc, T* __restrict__ out, CornerSpec cs,
                               int64_t N, int first) {
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < N;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = f, idx = 0;
    bool ok = true;
#pragma unroll
    for (int a = 2; a >= 0; --a) {
      if (a >= cs.d) continue;
      const int64_t x = r % cs.ext[a];
      r /= cs.ext[a];
      const int64_t t = (cs.far >> a) & 1 ? x + cs.k[a] : x;
      int64_t src;
      if ((cs.suffix >> a) & 1) {
        ok = ok && t < cs.ext[a];
        src = t;
      } else {
        ok = ok && t >= 1;
        src = t - 1 < cs.ext[a] - 1 ? t - 1 : cs.ext[a] - 1;
      }
      idx += src * cs.str[a];
    }
    if (first) {
      const T id = Op::template identity<T>();
      st1(out + f, ok ? Op::apply(id, sc[idx]) : id);
    } else if (ok) {
      out[f] = Op::apply(out[f], sc[idx]);
    }
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

template <class T, class Op>
int go_scan(const T* in, T* out, int64_t outer, int64_t n, int64_t inner, int64_t L, int64_t nseg,
            int rev, cudaStream_t s) {
  if (inner == 1) {
    constexpr int WARPS = 4;
    const int64_t groups = (outer * nseg + 31) / 32;
    if constexpr (sizeof(T) == 4) {
      k_scan_rows<T, Op, WARPS, 64><<<(unsigned)grid_for(groups * 32, WARPS * 32, 16),
                                      WARPS * 32, 0, s>>>(in, out, outer, n, L, nseg, rev);
    } else {
      k_scan_rows<T, Op, WARPS, 32><<<(unsigned)grid_for(groups * 32, WARPS * 32, 16),
                                      WARPS * 32, 0, s>>>(in, out, outer, n, L, nseg, rev);
    }
    return 1;
  }
  constexpr int VE = 16 / sizeof(T);
  const bool vec = inner % VE == 0 && ((uintptr_t)in % 16) == 0 && ((uintptr_t)out % 16) == 0;
  const int64_t want = (int64_t)num_sms() * 1024;
  if (vec && outer * (inner / VE) * nseg >= want) {
    const int64_t work = outer * (inner / VE) * nseg;
    k_scan_strided<T, Op, VE, 8><<<(unsigned)grid_for(work, 256, 8), 256, 0, s>>>(
        in, out, outer, n, inner, L, nseg, rev);
  } else {
    // few lines: one element per thread (VE-fold more threads) and 16 rows
    // of loads in flight to cover the latency of the sequential walk
    const int64_t work = outer * inner * nseg;
    k_scan_strided<T, Op, 1, 16><<<(unsigned)grid_for(work, 256, 8), 256, 0, s>>>(
        in, out, outer, n, inner, L, nseg, rev);
  }
  return 1;
}

template <class T>
int go_query(const T* S, T* out, const QShape& q, int64_t N, const void* total, int mode,
             const FastMod& fm, cudaStream_t s) {
  typedef typename AccOf<T>::type Acc;
  const Acc* tot = (const Acc*)total;
  constexpr int VE = 16 / sizeof(T);
  if (q.d >= 2 && q.d <= 6 && q.ext[q.d - 1] >= 512 && q.ext[q.d - 1] % VE == 0 &&
      ((uintptr_t)S % 16) == 0) {
    const int64_t n = q.ext[q.d - 1];
    const int NQ = 1 << (q.d - 2);
    const size_t smem = (size_t)4 * NQ * (n + VE) * sizeof(T);
    if (smem <= 96 * 1024) {
      const int64_t chains = N / n / q.ext[q.d - 2] * q.k[q.d - 2];
      // many chains: 128-thread CTAs (8 outputs of a 1024-wide row per thread
      // per step amortise the step's staging and ring bookkeeping), at most 4
      // per SM (more concurrent chains spread the shared S planes past L2:
      // C4 f32 query 2.24 -> 1.69 ms, C5 f64 0.48 -> 0.435 ms); few chains:
      // 256 threads each
      const int tpb = chains >= 2 * (int64_t)num_sms() ? 128 : 256;
      int per_sm = (int)((200 * 1024) / smem);
      per_sm = per_sm < 1 ? 1 : per_sm > 4 ? 4 : per_sm;
      const int64_t cap = (int64_t)num_sms() * per_sm;
      // equal chain counts per CTA: the fewest CTAs that keep the same rounds
      const int64_t rounds = (chains + cap - 1) / cap;
      const unsigned gr = (unsigned)((chains + rounds - 1) / rounds);
#define EXSUM_CHAIN_N(DH, NT)                                                                  \
  {                                                                                            \
    if (tpb == 128) {                                                                          \
      auto kfn = k_sat_query_chain<T, DH, NT, 128>;                                            \
      ensure_smem((const void*)kfn, smem);                                                     \
      kfn<<<gr, 128, smem, s>>>(S, out, q, chains, tot, mode, fm);                             \
    } else {                                                                                   \
      auto kfn = k_sat_query_chain<T, DH, NT, 256>;                                            \
      ensure_smem((const void*)kfn, smem);                                                     \
      kfn<<<gr, 256, smem, s>>>(S, out, q, chains, tot, mode, fm);                             \
    }                                                                                          \
  }
#define EXSUM_CHAIN(DH)                                                                        \
  {                                                                                            \
    if (n == 512) EXSUM_CHAIN_N(DH, 512)                                                       \
    else if (n == 1024) EXSUM_CHAIN_N(DH, 1024)                                                \
    else EXSUM_CHAIN_N(DH, 0)                                                                  \
  }
      switch (q.d) {
        case 2: EXSUM_CHAIN(1) break;
        case 3: EXSUM_CHAIN(2) break;
        case 4: EXSUM_CHAIN(3) break;
        case 5: EXSUM_CHAIN(4) break;
        case 6: EXSUM_CHAIN(5) break;
      }
#undef EXSUM_CHAIN
#undef EXSUM_CHAIN_N
      return 1;
    }
  }
  if (q.d >= 2 && q.d <= 6 && q.ext[q.d - 1] < (1LL << 30)) {
    const int64_t n = q.ext[q.d - 1];
    const int64_t rows = N / n;
    int G = 1;  // lanes per row: each handles 4 x values per step (XU)
    while (G < 32 && 4 * G < n) G *= 2;
    const int64_t warps = (rows + (32 / G) - 1) / (32 / G);
    const unsigned gr = (unsigned)grid_for(warps * 32, 256, 8);
    switch (q.d) {
      case 2: k_sat_query_rows<T, 1><<<gr, 256, 0, s>>>(S, out, q, rows, G, tot, mode, fm); break;
      case 3: k_sat_query_rows<T, 2><<<gr, 256, 0, s>>>(S, out, q, rows, G, tot, mode, fm); break;
      case 4: k_sat_query_rows<T, 3><<<gr, 256, 0, s>>>(S, out, q, rows, G, tot, mode, fm); break;
      case 5: k_sat_query_rows<T, 4><<<gr, 256, 0, s>>>(S, out, q, rows, G, tot, mode, fm); break;
      case 6: k_sat_query_rows<T, 5><<<gr, 256, 0, s>>>(S, out, q, rows, G, tot, mode, fm); break;
    }
    return 1;
  }
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

int launch_scan(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                int64_t inner, int64_t L, int64_t nseg, int rev, cudaStream_t s) {
  if (op == 1) {
    if (dtype != 2) return -1;
    return go_scan<i64, OpMax>((const i64*)in, (i64*)out, outer, n, inner, L, nseg, rev, s);
  }
  switch (dtype) {
    case 0: return go_scan<float, OpAdd>((const float*)in, (float*)out, outer, n, inner, L, nseg, rev, s);
    case 1: return go_scan<double, OpAdd>((const double*)in, (double*)out, outer, n, inner, L, nseg, rev, s);
    case 2: return go_scan<i64, OpAdd>((const i64*)in, (i64*)out, outer, n, inner, L, nseg, rev, s);
  }
  return -1;
}

int launch_seg_carry(int dtype, int op, void* out, void* tot, int64_t outer, int64_t n,
                     int64_t inner, int64_t L, int64_t nseg, int rev, int step, cudaStream_t s) {
  const int64_t work = step == 0 ? outer * (nseg - 1) * inner : outer * (n - L) * inner;
  const unsigned g = (unsigned)grid_for(work, 256, 8);
#define EXSUM_SEG(T, OP)                                                                        \
  if (step == 0)                                                                                \
    k_seg_gather<T><<<g, 256, 0, s>>>((const T*)out, (T*)tot, outer, n, inner, L, nseg, rev);   \
  else                                                                                          \
    k_carry_add<T, OP><<<g, 256, 0, s>>>((T*)out, (const T*)tot, outer, n, inner, L, nseg, rev); \
  return 1;
  if (op == 1) {
    if (dtype != 2) return -1;
    EXSUM_SEG(i64, OpMax)
  }
  switch (dtype) {
    case 0: { EXSUM_SEG(float, OpAdd) }
    case 1: { EXSUM_SEG(double, OpAdd) }
    case 2: { EXSUM_SEG(i64, OpAdd) }
  }
#undef EXSUM_SEG
  return -1;
}

int launch_corner_apply(int dtype, int op, const void* sc, void* out, const CornerSpec& cs,
                        int64_t N, int first, cudaStream_t s) {
  const unsigned g = (unsigned)grid_for(N, 256, 8);
  if (op == 1) {
    if (dtype != 2) return -1;
    k_corner_apply<i64, OpMax><<<g, 256, 0, s>>>((const i64*)sc, (i64*)out, cs, N, first);
    return 1;
  }
  switch (dtype) {
    case 0: k_corner_apply<float, OpAdd><<<g, 256, 0, s>>>((const float*)sc, (float*)out, cs, N, first); return 1;
    case 1: k_corner_apply<double, OpAdd><<<g, 256, 0, s>>>((const double*)sc, (double*)out, cs, N, first); return 1;
    case 2: k_corner_apply<i64, OpAdd><<<g, 256, 0, s>>>((const i64*)sc, (i64*)out, cs, N, first); return 1;
  }
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
