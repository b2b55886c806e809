// exsum_launch.h -- host-side launchers shared by the C-ABI orchestration.
//
// Every launcher works on a 3-D view [outer, n, inner] of a C-order array
// (outer = prod of extents before the axis, inner = prod after it), which is
// how windowed_sum_axis (scan.py:61-102) sees any axis of any d.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace exsum {

enum DType { F32 = 0, F64 = 1, I64 = 2 };
enum OpCode { ADD = 0, MAX = 1 };

// One windowed pass along the middle axis of [outer, n, inner]:
// out[o, x, i] = (+)_{y in [x, min(x+k, n))} in[o, y, i], with the reference's
// exact association (in-block right-nested suffix, left-nested prefix, one
// stitch combine).  in != out.  `total` (device, nullable) turns on the BDBSC
// complement epilogue out = total (-) value (float32 data: total is a double).
// Returns the number of kernels launched.
// Optional work piggy-backed on a strided pass over the raw input:
//   kind 1: per-warp row partials of the last axis (row_len elements per row)
//           into buf; on success ppr = partials per row (finish with
//           launch_rowpart_final);
//   kind 2: per-CTA partial totals into buf (capacity cap); on success ppr =
//           number of partials (finish with launch_total_final).
// n_out >= 0: produce only rows [0, n_out) along the axis (the output has
// n_out rows; outer must be 1) -- a shard reading a halo beyond its planes;
// n_out_done reports whether the launched kernel honoured it.
struct PassExtra {
  int kind = 0;
  void* buf = nullptr;
  int64_t row_len = 0;
  int64_t cap = 0;
  int done = 0;
  int64_t ppr = 0;
  int64_t n_out = -1;
  int n_out_done = 0;
};

int launch_pass(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                int64_t inner, int64_t k, const void* total, cudaStream_t s,
                PassExtra* ex = nullptr);
int launch_rowpart_final(int dtype, int op, const void* part, void* R, int64_t rows, int64_t ppr,
                         cudaStream_t s);
int launch_total_final(int dtype, int op, const void* partials, int64_t np, void* total,
                       cudaStream_t s);

// Deterministic total fold of N elements into *total (device; double for
// float32).  partials: device scratch of reduce_partials_count() accumulators.
int reduce_partials_count();
int launch_total(int dtype, int op, const void* in, int64_t N, void* partials, void* total,
                 cudaStream_t s);

// BDBSC complement for a route with no windowed pass: out = total (-) in.
int launch_complement(int dtype, const void* in, void* out, int64_t N, const void* total,
                      cudaStream_t s);

// Box-complement tail of a 3-D array (tail2d.cu): R (n0 x n1) from row
// partials part[n0*n1][ppr] (or, part == nullptr, R as given), R2 (n0) its
// fold over the last axis, Tout = BC(R, (k0, k1)).  stage 0 writes R and R2,
// stage 1 (after it) writes Tout; one launch each.
int tail2d_ok(int dtype, int64_t n0, int64_t n1, int64_t k0);
int launch_tail2d(int dtype, int op, const void* part, int64_t ppr, void* R, void* R2, void* Tout,
                  int64_t n0, int64_t n1, int64_t k0, int64_t k1, cudaStream_t s, int stage);
// The tail of one axis-0 shard (sharded box-complement): stage 0 R2[i] = fold
// of R row i for the rows [gb, ge) held at R (local indexing); stage 1 the rows
// [gb, ge) of T = BC(R) from R2 (all n0 rows) and R's rows [gb, ge + k0 - 1)
// (the shard's own and its halo), R and Tout addressed by the global row.
int launch_tail2d_shard(int dtype, int op, const void* R, void* R2, void* Tout, int64_t n0,
                        int64_t n1, int64_t k0, int64_t k1, int64_t gb, int64_t ge, cudaStream_t s,
                        int stage);

// R[r] = (+)_x in[r, x] for rows of length n (box-complement reduction of the
// peeled last axis).
int launch_row_reduce(int dtype, int op, const void* in, void* R, int64_t rows, int64_t n,
                      cudaStream_t s);

// Box-complement round along the last axis (rows of length n):
// out[r, x] = P[r, x-1] (+) S[r, x+k] (+) T[r], with P/S the full-row
// inclusive prefix/suffix of W and T the tail (nullable = identity).  Terms
// out of range are the identity.  scratch: rows*n elements, used only when a
// row does not fit in shared memory.
int launch_excl_rows(int dtype, int op, const void* W, void* out, const void* T, int64_t rows,
                     int64_t n, int64_t k, void* scratch, cudaStream_t s);
size_t excl_rows_scratch_elems(int dtype, int64_t rows, int64_t n);

// Fused pass pair over [outer, n1, n2]: the windowed pass along n1 (window
// k1) followed by a row op along n2 -- ROW_WIN: windowed pass with window k2
// (+ BDBSC epilogue when total != nullptr); ROW_EXCL: box-complement round with
// shift k2 and tail T (nullable).  fused_pair_ok() decides eligibility.
enum { ROW_WIN = 0, ROW_EXCL = 1, ROW_EXCL_ADD = 2, ROW_EXCL_BLK = 3 /* 2, 3 internal: chosen by go_fused */ };
int fused_pair_ok(int dtype, int op, int64_t n2, int64_t k1, int64_t k2, int mode);
int launch_fused_pair(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n1,
                      int64_t n2, int64_t k1, int64_t k2, int mode, const void* total,
                      const void* Tail, cudaStream_t s);

// Box-complement for max as per-axis marginals (idem_max.cu): out[x] =
// (+)_a F_a[x_a], F_a the 1-D excluded window of the marginal M_a (the fold over
// every axis but a) -- exact for an idempotent operator.  idem_max_ok() decides
// eligibility (EXSUM_IDEM=0 disables); launch_idem_max(stage): -1 sizes the
// workspace only (*ws_bytes), 0 the marginals and tables (one read of A), 1 the
// broadcast (one write of out).
#define EXSUM_IDEM_MAX_DIMS 32
int idem_max_ok(int dtype, int op, int d, const int64_t* ext);
int launch_idem_max(int dtype, const void* in, void* out, int d, const int64_t* ext,
                    const int64_t* k, void* ws, size_t* ws_bytes, cudaStream_t st, int stage);
// A shard (global planes [x0, x0 + n_own) of axis 0; ext global): stage 0 the
// shard's marginals as plain values into marg (S = sum of ext), stage 1 the
// shard's output planes from the all-reduced marginals; -1 sizes ws.
int launch_idem_max_shard(int dtype, const void* in, void* out, void* marg, int d,
                          const int64_t* ext, const int64_t* k, int64_t x0, int64_t n_own,
                          void* ws, size_t* ws_bytes, cudaStream_t st, int stage);

// The last two windowed passes of BDBS (windows k1 == k2 == 32) in one launch
// over shared-memory tiles with their stitch halos (tile_pair.cu); total !=
// nullptr applies the BDBSC complement epilogue.  tile_pair_ok() decides
// eligibility (EXSUM_TILE_PAIR=0 disables; arrays of at most 64 MB: on larger
// ones the two streaming passes are faster).
int tile_pair_ok(int dtype, int op, int64_t N, int64_t n1, int64_t n2, int64_t k1, int64_t k2);
int launch_tile_pair(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n1,
                     int64_t n2, int64_t k1, int64_t k2, const void* total, cudaStream_t s);

// Trailing-block fusion (block_fused.cu): the windowed passes along the last m
// axes in one kernel when a block of those axes (last axis padded to an odd
// length) fits in shared memory.  block_fused_plan picks the largest such m
// (axes >= first_axis, at least two passes, windows 2/4/8/16) and returns 1.
#define BF_MAX 6
struct BlockSpec {
  int m = 0;
  int n[BF_MAX], k[BF_MAX], inner[BF_MAX];
  uint32_t magic_inner[BF_MAX];
  uint32_t magic_nl = 0;
  int64_t B = 0;    // elements per block
  int rowp = 0;     // padded row length
  int G = 1;        // blocks per CTA tile
  int K = 0;        // the window of every fused axis with a pass
  int threads = 256;
  size_t smem = 0;  // bytes per tile
};
int block_fused_plan(int dtype, int d, const int64_t* ext, const int64_t* k, int first_axis,
                     BlockSpec* out);
int launch_block_fused(int dtype, int op, const void* in, void* out, int64_t N, const BlockSpec& bs,
                       const void* total, cudaStream_t s);

// Two consecutive strided passes (axes a, a+1 of equal extent 16 or 28, one
// window) in one HBM round trip over [outer, na, nb, inner] (outer_pair.cu)
int outer_pair_ok(int dtype, int op, int64_t na, int64_t nb, int64_t inner, int64_t ka, int64_t kb);
int launch_outer_pair(int dtype, int op, const void* in, void* out, int64_t outer, int64_t na,
                      int64_t nb, int64_t inner, int64_t ka, int64_t kb, const void* total,
                      cudaStream_t s);

// L2-pipelined 3-D schedule (l2pipe.cu; opt-in EXSUM_L2PIPE=1): float32
// [n0, n1, 1024] with box 16^3 in one persistent kernel -- mode 0 bdbs,
// mode 1 the box-complement W passes + row round with tail T.
int l2pipe_ok(int dtype, int op, int d, const int64_t* ext, const int64_t* k);
size_t l2pipe_workspace_bytes(const int64_t* ext);
int launch_l2pipe(int mode, const void* in, void* out, const int64_t* ext, const void* Tail,
                  void* ws, cudaStream_t s);

// ---------------------------------------------- sat / satc / mod-add (sat.cu)

// Inclusive running fold (ops.accumulate: np.add / np.maximum .accumulate)
// along the middle axis of [outer, n, inner] -- reversed (suffix) when rev --
// restarted every L elements of the (possibly reversed) line (nseg segments;
// nseg == 1: plain sequential scan).  in == out is allowed.
int launch_scan(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                int64_t inner, int64_t L, int64_t nseg, int rev, cudaStream_t s);
// Segmented scans: step 0 gathers the segment totals into tot[outer, nseg-1,
// inner]; step 1 folds the scanned totals back in as carries.
int launch_seg_carry(int dtype, int op, void* out, void* tot, int64_t outer, int64_t n,
                     int64_t inner, int64_t L, int64_t nseg, int rev, int step, cudaStream_t s);

// One corner pattern's contribution into out (first: out = identity (+) it).
struct CornerSpec {
  int d;
  int64_t ext[3], k[3], str[3];
  int suffix;  // bit a: axis a is a suffix (S) letter
  int far;     // bit a: the threshold is the far face x + k
};
int launch_corner_apply(int dtype, int op, const void* sc, void* out, const CornerSpec& cs,
                        int64_t N, int first, cudaStream_t s);

#define EXSUM_QMAX 32
struct QShape {
  int d;
  int64_t ext[EXSUM_QMAX];
  int64_t k[EXSUM_QMAX];
  int64_t str[EXSUM_QMAX];
};
enum { QUERY_PLAIN = 0, QUERY_COMPLEMENT = 1, QUERY_MOD = 2, QUERY_MOD_COMPLEMENT = 3 };

// floor modulus by a runtime m in [2, 2^31]: inv = floor((2^64 - 1) / m).
struct FastMod {
  unsigned long long m;
  unsigned long long inv;
};
inline FastMod make_fastmod(int64_t m) {
  FastMod f;
  f.m = (unsigned long long)(m > 1 ? m : 2);
  f.inv = ~0ULL / f.m;
  return f;
}

// out = the 2^d-corner query of the running-sum table S (included.py:98-121)
// with the route epilogue `mode` (total: Acc* for QUERY_COMPLEMENT, int64*
// for QUERY_MOD_COMPLEMENT).
int launch_sat_query(int dtype, const void* S, void* out, const QShape& q, int64_t N,
                     const void* total, int mode, const FastMod& fm, cudaStream_t s);

// mod-add element maps on int64: mode 0 out = in mod m (in may equal out);
// mode 1 out = ((total mod m) - in) mod m.
int launch_mod_map(const void* in, void* out, int64_t N, int mode, const FastMod& fm,
                   const void* total, cudaStream_t s);

struct SliceSpec {
  int d;
  int64_t ext[EXSUM_QMAX];
  int fixed[EXSUM_QMAX];
};
// out[x] = in[x] for x with x_j = n_j - 1 on every fixed axis (count = the
// product of the free extents).
int launch_copy_slice(const void* in, void* out, const SliceSpec& sp, int64_t count,
                      cudaStream_t s);

// ------------------------------------------------ building blocks (pieces.cu)
// op: 0 add, 1 max (int64), 2 mod-add (int64, fm)
int launch_add_contribution(int dtype, int op, const FastMod& fm, const void* src, void* dst,
                            int64_t outer, int64_t n, int64_t inner, int64_t offset,
                            cudaStream_t s);
// kind 0 combine_into, 1 subtract_into, 2 rsubtract_scalar (scalar read from host)
int launch_elementwise(int dtype, int op, const FastMod& fm, void* dst, const void* src,
                       const void* scalar_host, int kind, int64_t n, cudaStream_t s);
int launch_fold_result(int dtype, int op, const FastMod& fm, const void* acc, void* out,
                       cudaStream_t s);

size_t dtype_size(int dtype);
int num_sms();

// Segments per line for the streaming kernels (one CTA streams one (line,
// segment) item of `nunits` units).  With one resident CTA per SM the count
// minimises (waves of items, rounded up) x (units per item + 1 for the halo
// block and pipeline fill): a whole extra wave for a few leftover items costs
// more than a short halo (C5 f64: 512 single-line items on 148 SMs were 3.46
// waves).  Smaller CTAs keep ~3 waves of items so several stay resident per SM.
inline int64_t pick_segments(int64_t lines, int64_t nunits, int per_sm) {
  const int64_t slots = (int64_t)num_sms() * per_sm;
  // segments of >= 4 units bound the halo re-reads; an array too small to
  // fill the machine that way (the box-complement tail levels: one 1024-row
  // line) takes segments down to one unit
#ifndef EXSUM_SMALL_SEG
#define EXSUM_SMALL_SEG 1
#endif
  int64_t max_seg = (EXSUM_SMALL_SEG && lines * (nunits / 4) < slots) ? nunits : nunits / 4;
  if (max_seg < 1) max_seg = 1;
  if (per_sm > 1) {
    int64_t nseg = (slots * 3 + lines - 1) / lines;
    if (nseg > max_seg) nseg = max_seg;
    return nseg < 1 ? 1 : nseg;
  }
  if (max_seg > 64) max_seg = 64;
  int64_t nseg = 1;
  double best = 1e300;
  for (int64_t c = 1; c <= max_seg; ++c) {
    const int64_t per = (nunits + c - 1) / c;
    const int64_t items = lines * ((nunits + per - 1) / per);
    const double cost = (double)((items + slots - 1) / slots) * ((double)per + 1.0);
    if (cost < best * 0.999) {
      best = cost;
      nseg = c;
    }
  }
  return nseg;
}

}  // namespace exsum
