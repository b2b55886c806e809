// exsum_capi.cu -- C ABI (include/exsum_b200.h) and route orchestration.
//
// Routes (reference pkg/src/exsum):
//   bdbs            included.py:124-129   one windowed pass per axis, axes in
//                                          order 0..d-1 (bit-exact association)
//   bdbsc           excluded.py:88-90     total fold + bdbs, complement fused
//                                          into the last pass's stores
//   box-complement  excluded.py:129-159   slab decomposition, peeling the LAST
//                                          axis first (see below)
//   sat / satc      included.py:37-121,   running-sum table (d sequential
//                   excluded.py:83-85     scans) + one 2^d-corner query (sat.cu)
//   corners         excluded.py:191-292   2^d scanned copies (P/S per axis) and
//                                          their corner contributions (2-D, 3-D)
//   mod-add:<m>     monoid.py:235-286     any route: canonical residues, the
//                                          exact int64 + route, a mod-m epilogue
//
// Box-complement order.  The reference peels dimension 0 first: round i adds
// the "below"/"above" slabs of dimension i on the reduced slice.  The slab
// decomposition is valid in any dimension order (the complement of a box is
// the disjoint union, over the peeled dimension, of {outside the window in
// that dimension, inside the box in the not-yet-peeled ones} plus the
// complement in the remaining dimensions of the reduction), so this build
// peels the contiguous last axis first:
//     BC(A, k) = E_{d-1}(W) (+) bcast_rows( BC(R, k[:-1]) )
//     W = windowed passes of A along axes 0..d-2 (same kernels as bdbs)
//     R = (+)-reduction of A over the last axis
//     E_{d-1}(W)[.., x] = P(W)[.., x-1] (+) S(W)[.., x+k_{d-1}]  (full-row scans)
// so the full-array rounds are d-1 streaming passes plus one row kernel, and
// the recursion runs on arrays n_{d-1} times smaller.  Integer + and max are
// exact, so the result is bit-identical to the reference; float + agrees to
// the reassociation bound.
#include <cuda_runtime.h>

#include <stdio.h>
#include <string.h>

extern char** environ;

#include <mutex>
#include <string>
#include <vector>

#include "../../include/exsum_b200.h"
#include "exsum_launch.h"

using namespace exsum;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(EXSUM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return EXSUM_OK;
}

// Optional per-launch CUDA-event profiler (exsum_profile_*): bench.py uses it
// to time each kernel on its own stream inside the timed region and to pair
// it with the kernel's algorithmic bytes for the roofline.
struct ProfRec {
  const char* name;
  double bytes;
  cudaEvent_t a, b;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};
thread_local Profiler g_prof;

struct ProfScope {
  cudaStream_t st;
  bool on;
  ProfScope(const char* name, double bytes, cudaStream_t s) : st(s), on(g_prof.on) {
    if (!on) return;
    ProfRec r{name, bytes, g_prof.ev(), g_prof.ev()};
    cudaEventRecord(r.a, st);
    g_prof.recs.push_back(r);
  }
  ~ProfScope() {
    if (on) cudaEventRecord(g_prof.recs.back().b, st);
  }
};

struct Shape {
  int d = 0;
  int64_t ext[EXSUM_MAX_DIMS];
  int64_t k[EXSUM_MAX_DIMS];
  int64_t N = 1;
};

// tensor.py:20-48 (validate_extents + normalize_box): arity, n >= 1, k >= 1,
// k clamped to n.
int normalize(int d, const int64_t* ext, const int64_t* box, Shape* s) {
  if (d < 1 || d > EXSUM_MAX_DIMS) return fail(EXSUM_EUSAGE, "extents must have 1..32 dimensions");
  if (!ext || !box) return fail(EXSUM_EUSAGE, "null extents or box");
  s->d = d;
  s->N = 1;
  for (int i = 0; i < d; ++i) {
    if (ext[i] < 1) return fail(EXSUM_EUSAGE, "every extent must be >= 1");
    if (box[i] < 1) return fail(EXSUM_EUSAGE, "every box side must be >= 1");
    s->ext[i] = ext[i];
    s->k[i] = box[i] < ext[i] ? box[i] : ext[i];
    s->N *= ext[i];
  }
  return EXSUM_OK;
}

int check_types(int dtype, int op, int64_t modulus = 0) {
  if (dtype != EXSUM_F32 && dtype != EXSUM_F64 && dtype != EXSUM_I64)
    return fail(EXSUM_ECONFIG, "unsupported dtype (float32, float64, int64)");
  if (op != EXSUM_ADD && op != EXSUM_MAX && op != EXSUM_MODADD)
    return fail(EXSUM_ECONFIG, "unsupported operator");
  if (op == EXSUM_MAX && dtype != EXSUM_I64)
    return fail(EXSUM_ECONFIG, "max is provided for int64 only (max-i64, monoid.py:207-232)");
  if (op == EXSUM_MODADD) {
    if (dtype != EXSUM_I64) return fail(EXSUM_ECONFIG, "mod-add is an int64 monoid (monoid.py:235-248)");
    // ModAddOps.__init__ (monoid.py:250-256): 2 <= m <= 2^31
    if (modulus < 2 || modulus > ((int64_t)1 << 31))
      return fail(EXSUM_ECONFIG, "mod-add modulus must be in [2, 2147483648]");
  }
  return EXSUM_OK;
}

// Bump allocator over the caller's workspace; base == nullptr sizes only.
struct Arena {
  char* base;
  size_t off = 0;
  explicit Arena(void* b) : base((char*)b) {}
  void* take(size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    void* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
};

// The fused pass pair moves 16-byte vectors; a caller's array off that
// alignment (a view into a larger buffer) takes the unfused kernels instead.
bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

int64_t prod(const int64_t* e, int lo, int hi) {
  int64_t p = 1;
  for (int i = lo; i < hi; ++i) p *= e[i];
  return p;
}

// Windowed passes along the listed axes, ending in `final_dst`; intermediate
// results alternate between final_dst and `other` (both != src).
struct PassPlan {
  int axes[EXSUM_MAX_DIMS];
  int count = 0;
};

PassPlan plan_passes(const Shape& s, int upto) {
  PassPlan p;
  for (int a = 0; a < upto; ++a)
    if (s.k[a] > 1) p.axes[p.count++] = a;
  return p;
}

// One windowed pass along axis a (profiled), optionally piggy-backing a
// reduction over the raw input (PassExtra).
int one_pass(const Shape& s, int a, int dtype, int op, const void* src, void* dst,
             const void* epi_total, cudaStream_t st, int* launches, PassExtra* ex) {
  const size_t es = dtype_size(dtype);
  ProfScope ps(a == s.d - 1 ? "pass_rows" : "pass_strided", 2.0 * (double)s.N * es, st);
  int rc = launch_pass(dtype, op, src, dst, prod(s.ext, 0, a), s.ext[a], prod(s.ext, a + 1, s.d),
                       s.k[a], epi_total, st, ex);
  if (rc < 0) return fail(EXSUM_ECONFIG, "no kernel for this dtype/operator");
  *launches += rc;
  return EXSUM_OK;
}

// Passes along p.axes, the first reading src, the last writing final_dst,
// intermediates alternating with `other`.  after_first() runs (in both the
// sizing and the launch pass) right after the first pass is enqueued.
template <class F>
int run_chain(const Shape& s, const PassPlan& p, int dtype, int op, const void* src,
              void* final_dst, void* other, const void* epi_total, cudaStream_t st,
              int* launches, bool live, PassExtra* ex0, F after_first) {
  // steps: one pass, or two consecutive small strided axes as one outer pair
  // (outer_pair.cu) when every buffer of the chain is 16-byte aligned
  const size_t es = dtype_size(dtype);
  const bool al = aligned16(src) && aligned16(final_dst) && (!other || aligned16(other));
  int first[EXSUM_MAX_DIMS], len[EXSUM_MAX_DIMS], nsteps = 0;
  for (int i = 0; i < p.count;) {
    const int a = p.axes[i];
    const bool pair = al && i + 1 < p.count && p.axes[i + 1] == a + 1 && a + 2 < s.d &&
                      !(i == 0 && ex0) &&
                      outer_pair_ok(dtype, op, s.ext[a], s.ext[a + 1], prod(s.ext, a + 2, s.d),
                                    s.k[a], s.k[a + 1]);
    first[nsteps] = i;
    len[nsteps++] = pair ? 2 : 1;
    i += pair ? 2 : 1;
  }
  const void* cur = src;
  for (int j = 0; j < nsteps; ++j) {
    const int remaining = nsteps - 1 - j;
    void* dst = (remaining % 2 == 0) ? final_dst : other;
    const int i = first[j];
    if (live) {
      const void* epi = j == nsteps - 1 ? epi_total : nullptr;
      if (len[j] == 2) {
        const int a = p.axes[i];
        ProfScope ps("outer_pair", 2.0 * (double)s.N * es, st);
        const int rc = launch_outer_pair(dtype, op, cur, dst, prod(s.ext, 0, a), s.ext[a],
                                         s.ext[a + 1], prod(s.ext, a + 2, s.d), s.k[a], s.k[a + 1],
                                         epi, st);
        if (rc <= 0) return fail(EXSUM_ECUDA, "outer pass pair failed to launch");
        *launches += rc;
      } else {
        int rc = one_pass(s, p.axes[i], dtype, op, cur, dst, epi, st, launches,
                          i == 0 ? ex0 : nullptr);
        if (rc) return rc;
      }
    }
    if (j == 0) {
      int rc = after_first();
      if (rc) return rc;
    }
    cur = dst;
  }
  return EXSUM_OK;
}

int no_hook() { return EXSUM_OK; }

// ------------------------------------------------------------------ routes --

int route_bdbs(const Shape& s, int dtype, int op, const void* in, void* out, Arena& ar,
               bool complement, cudaStream_t st, int* launches,
               const void* given_total = nullptr) {
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  PassPlan p = plan_passes(s, s.d);
  void* partials = nullptr;
  void* total = nullptr;
  if (complement) {
    partials = ar.take((size_t)reduce_partials_count() * 8);
    total = ar.take(8);
  }
  void* other = p.count >= 2 ? ar.take((size_t)s.N * es) : nullptr;
  if (given_total) total = const_cast<void*>(given_total);  // shard: the global total
  auto full_total = [&]() {
    if (live && !given_total) {
      ProfScope ps("total", (double)s.N * es, st);
      *launches += launch_total(dtype, op, in, s.N, partials, total, st);
    }
  };
  if (p.count == 0) {
    if (complement) full_total();
    if (!live) return EXSUM_OK;
    ProfScope ps(complement ? "complement" : "copy", 2.0 * (double)s.N * es, st);
    if (complement) {
      *launches += launch_complement(dtype, in, out, s.N, total, st);
    } else {
      cudaMemcpyAsync(out, in, (size_t)s.N * es, cudaMemcpyDeviceToDevice, st);
    }
    return EXSUM_OK;
  }
  const int d = s.d;
  if (!complement && l2pipe_ok(dtype, op, d, s.ext, s.k) && aligned16(in) && aligned16(out)) {
    void* ws = ar.take(l2pipe_workspace_bytes(s.ext));
    if (live) {
      ProfScope ps("l2pipe", 2.0 * (double)s.N * es, st);
      const int rc = launch_l2pipe(0, in, out, s.ext, nullptr, ws, st);
      if (rc < 0) return fail(EXSUM_ECUDA, "L2-pipelined kernel failed to launch");
      *launches += rc;
    }
    return EXSUM_OK;
  }
  const bool fused = p.count >= 2 && p.axes[p.count - 2] == d - 2 && p.axes[p.count - 1] == d - 1 &&
                     fused_pair_ok(dtype, op, s.ext[d - 1], s.k[d - 2], s.k[d - 1], ROW_WIN) &&
                     aligned16(out) && (p.count > 2 || aligned16(in));
  // windows the fused pair has no template for (k = 32) on small arrays: the
  // last two passes as one tiled kernel (tile_pair.cu)
  const bool tilep = !fused && p.count >= 2 && p.axes[p.count - 2] == d - 2 &&
                     p.axes[p.count - 1] == d - 1 &&
                     tile_pair_ok(dtype, op, s.N, s.ext[d - 2], s.ext[d - 1], s.k[d - 2],
                                  s.k[d - 1]) &&
                     aligned16(out) && (p.count > 2 || aligned16(in));
  PassPlan head = p;
  if (fused || tilep) head.count -= 2;
  // otherwise the trailing axes as one shared-memory block when it fits
  // (block_fused.cu): the passes along axes >= d - m in one HBM round trip
  BlockSpec bsp;
  const bool blockf =
      !fused && !tilep && p.count >= 2 && block_fused_plan(dtype, d, s.ext, s.k, 0, &bsp);
  if (blockf) {
    head.count = 0;
    while (head.count < p.count && p.axes[head.count] < d - bsp.m) ++head.count;
  }
  // BDBSC total: folded into the first pass when a later pass applies it
  PassExtra ex0;
  ex0.kind = 2;
  ex0.buf = partials;
  ex0.cap = reduce_partials_count();
  const bool piggy =
      complement && !given_total && head.count >= 1 && (fused || tilep || blockf || head.count >= 2);
  if (complement && !piggy) full_total();
  auto finish_total = [&]() -> int {
    if (piggy && live) {
      if (ex0.done) {
        *launches += launch_total_final(dtype, op, partials, ex0.ppr, total, st);
      } else {
        full_total();
      }
    }
    return EXSUM_OK;
  };
  const void* mid = in;
  if (head.count > 0) {
    const bool tail_kernel = fused || tilep || blockf;
    void* head_dst = tail_kernel ? other : out;
    void* head_other = tail_kernel ? out : other;
    int rc = run_chain(s, head, dtype, op, in, head_dst, head_other, tail_kernel ? nullptr : total,
                       st, launches, live, piggy ? &ex0 : nullptr, finish_total);
    if (rc) return rc;
    mid = head_dst;
  }
  if (blockf && live) {
    ProfScope ps("block_fused", 2.0 * (double)s.N * es, st);
    int rc = launch_block_fused(dtype, op, mid, out, s.N, bsp, total, st);
    if (rc < 0) return fail(EXSUM_ECONFIG, "no block kernel for this dtype/operator");
    *launches += rc;
  }
  if (tilep && live) {
    ProfScope ps("tile_pair", 2.0 * (double)s.N * es, st);
    const int64_t n1 = s.ext[d - 2], n2 = s.ext[d - 1];
    int rc = launch_tile_pair(dtype, op, mid, out, s.N / (n1 * n2), n1, n2, s.k[d - 2], s.k[d - 1],
                              total, st);
    if (rc < 0) return fail(EXSUM_ECUDA, "tiled pass pair failed to launch");
    *launches += rc;
  }
  if (fused && live) {
    ProfScope ps("fused_pair", 2.0 * (double)s.N * es, st);
    const int64_t n1 = s.ext[d - 2], n2 = s.ext[d - 1];
    int rc = launch_fused_pair(dtype, op, mid, out, s.N / (n1 * n2), n1, n2, s.k[d - 2],
                               s.k[d - 1], ROW_WIN, total, nullptr, st);
    if (rc < 0) return fail(EXSUM_ECUDA, "fused pass pair failed to launch");
    *launches += rc;
  }
  return EXSUM_OK;
}

// The box-complement round after R/T are known: W passes along `head` (the
// first one may carry the R reduction, ex0, with hook() right after it),
// then the row round with tail T, fused with the last W pass when `fused`.
template <class F>
int bc_finish(const Shape& s, int dtype, int op, const void* src, void* dst, const void* T,
              const PassPlan& head, bool fused, PassExtra* ex0, F hook, Arena& ar,
              cudaStream_t st, int* launches) {
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  const int d = s.d;
  const int64_t n = s.ext[d - 1];
  const int64_t rows = s.N / n;
  const void* W = src;
  if (head.count > 0) {
    void* wbuf = ar.take((size_t)s.N * es);
    // the chain ends in wbuf; dst serves as the ping-pong partner
    int rc = run_chain(s, head, dtype, op, src, wbuf, dst, nullptr, st, launches, live, ex0,
                       hook);
    if (rc) return rc;
    W = wbuf;
  } else {
    int rc = hook();
    if (rc) return rc;
  }
  if (fused) {
    // last W pass (axis d-2) fused with the row round (fused_pair.cu)
    if (live) {
      ProfScope ps("fused_pair", (double)(2 * s.N + rows) * es, st);
      const int64_t n1 = s.ext[d - 2];
      int rc = launch_fused_pair(dtype, op, W, dst, s.N / (n1 * n), n1, n, s.k[d - 2], s.k[d - 1],
                                 ROW_EXCL, nullptr, T, st);
      if (rc < 0) return fail(EXSUM_ECUDA, "fused pass pair failed to launch");
      *launches += rc;
    }
    return EXSUM_OK;
  }
  void* scratch = ar.take(excl_rows_scratch_elems(dtype, rows, n) * es);
  if (live) {
    ProfScope ps("excl_rows", (double)(2 * s.N + rows) * es, st);
    *launches += launch_excl_rows(dtype, op, W, dst, T, rows, n, s.k[d - 1], scratch, st);
  }
  return EXSUM_OK;
}

// BC(src) -> dst, peeling the last axis (see file header).
int route_box_complement(const Shape& s, int dtype, int op, const void* src, void* dst,
                         Arena& ar, cudaStream_t st, int* launches) {
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  const int d = s.d;
  const int64_t n = s.ext[d - 1];
  const int64_t rows = s.N / n;
  if (idem_max_ok(dtype, op, d, s.ext)) {
    // max is idempotent: the per-axis marginal form (idem_max.cu), one read
    // and one write of the array
    size_t bytes = 0;
    launch_idem_max(dtype, src, dst, d, s.ext, s.k, nullptr, &bytes, st, -1);
    void* ws = ar.take(bytes);
    if (!live) return EXSUM_OK;
    static const char* names[2] = {"idem_scan", "idem_bcast"};
    for (int stage = 0; stage < 2; ++stage) {
      const double b = (double)s.N * es;
      ProfScope ps(names[stage], b, st);
      const int rc = launch_idem_max(dtype, src, dst, d, s.ext, s.k, ws, nullptr, st, stage);
      if (rc < 0) return fail(EXSUM_ECONFIG, "no marginal kernel for this dtype");
      *launches += rc;
    }
    return EXSUM_OK;
  }
  if (d == 1) {
    void* scratch = ar.take(excl_rows_scratch_elems(dtype, 1, n) * es);
    if (live) {
      ProfScope ps("excl_rows", 2.0 * (double)n * es, st);
      *launches += launch_excl_rows(dtype, op, src, dst, nullptr, 1, n, s.k[0], scratch, st);
    }
    return EXSUM_OK;
  }
  void* R = ar.take((size_t)rows * es);
  void* T = ar.take((size_t)rows * es);
  PassPlan p = plan_passes(s, d - 1);  // W = windowed passes along axes 0..d-2
  if (l2pipe_ok(dtype, op, d, s.ext, s.k) && aligned16(src) && aligned16(dst)) {
    // R needs all of A before any output row: a reduction pre-pass, the tail
    // T = BC(R, k[:-1]), then the W passes + row round in one persistent kernel
    if (live) {
      ProfScope ps("row_reduce", (double)(s.N + rows) * es, st);
      *launches += launch_row_reduce(dtype, op, src, R, rows, n, st);
    }
    Shape t;
    t.d = d - 1;
    t.N = rows;
    for (int i = 0; i < d - 1; ++i) {
      t.ext[i] = s.ext[i];
      t.k[i] = s.k[i];
    }
    int rc = route_box_complement(t, dtype, op, R, T, ar, st, launches);
    if (rc) return rc;
    void* ws = ar.take(l2pipe_workspace_bytes(s.ext));
    if (live) {
      ProfScope ps("l2pipe", (double)(2 * s.N + rows) * es, st);
      rc = launch_l2pipe(1, src, dst, s.ext, T, ws, st);
      if (rc < 0) return fail(EXSUM_ECUDA, "L2-pipelined kernel failed to launch");
      *launches += rc;
    }
    return EXSUM_OK;
  }
  const bool fused = p.count > 0 && p.axes[p.count - 1] == d - 2 &&
                     fused_pair_ok(dtype, op, n, s.k[d - 2], s.k[d - 1], ROW_EXCL) &&
                     aligned16(dst) && (p.count > 1 || aligned16(src));
  PassPlan head = p;
  if (fused) head.count -= 1;
  // R = reduction over the last axis, folded into the first W pass when
  // there is one (it reads the raw input anyway); then T = BC(R, k[:-1])
  PassExtra ex0;
  ex0.kind = 1;
  ex0.row_len = n;
  ex0.buf = head.count > 0 ? ar.take((size_t)(s.N / 32 + 1) * es) : nullptr;
  Shape t;
  t.d = d - 1;
  t.N = rows;
  for (int i = 0; i < d - 1; ++i) {
    t.ext[i] = s.ext[i];
    t.k[i] = s.k[i];
  }
  auto reduce_and_tail = [&]() -> int {
    if (d == 3 && tail2d_ok(dtype, s.ext[0], s.ext[1], s.k[0])) {
      // R is 2-D: R (from the row partials), its fold R2 and T = BC(R) in
      // two launches (tail2d.cu)
      void* R2 = ar.take((size_t)s.ext[0] * es);
      if (!live) return EXSUM_OK;
      if (!ex0.done) {
        ProfScope ps("row_reduce", (double)(s.N + rows) * es, st);
        *launches += launch_row_reduce(dtype, op, src, R, rows, n, st);
      }
      for (int stage = 0; stage < 2; ++stage) {
        ProfScope ps(stage ? "tail_group" : "tail_rows",
                     (double)(stage ? 2 : (ex0.done ? ex0.ppr + 1 : 1)) * rows * es, st);
        const int rc = launch_tail2d(dtype, op, ex0.done ? ex0.buf : nullptr, ex0.ppr, R, R2, T,
                                     s.ext[0], s.ext[1], s.k[0], s.k[1], st, stage);
        if (rc < 0) return fail(EXSUM_ECONFIG, "no tail kernel for this dtype/operator");
        *launches += rc;
      }
      return EXSUM_OK;
    }
    if (live) {
      if (ex0.done) {
        *launches += launch_rowpart_final(dtype, op, ex0.buf, R, rows, ex0.ppr, st);
      } else {
        ProfScope ps("row_reduce", (double)(s.N + rows) * es, st);
        *launches += launch_row_reduce(dtype, op, src, R, rows, n, st);
      }
    }
    return route_box_complement(t, dtype, op, R, T, ar, st, launches);
  };
  return bc_finish(s, dtype, op, src, dst, T, head, fused, &ex0, reduce_and_tail, ar, st, launches);
}

// Running sum along the middle axis of [outer, n, inner] (np.add.accumulate),
// src -> dst (in place allowed).  Lines are scanned sequentially (numpy's
// association) unless there are too few of them to fill the GPU; then the
// axis is cut into segments: local scans, an (in-place, recursive) scan of
// the segment totals, and a carry pass.
int scan_view(int dtype, const void* src, void* dst, int64_t outer, int64_t n, int64_t inner,
              Arena& ar, cudaStream_t st, int* launches, int op = EXSUM_ADD, int rev = 0) {
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  const int64_t ve = (int64_t)(16 / es);
  const int64_t lanes = inner == 1 ? outer : outer * (inner % ve == 0 ? inner / ve : inner);
  const int64_t want = (int64_t)num_sms() * 256;
  int64_t L = n, nseg = 1;
  if (lanes < want && n >= 4096) {
    nseg = (want + lanes - 1) / lanes;
    if (nseg > n / 1024) nseg = n / 1024;
    L = ((n + nseg - 1) / nseg + 31) / 32 * 32;
    nseg = (n + L - 1) / L;
  }
  if (live) {
    ProfScope ps(inner == 1 ? "sat_scan_rows" : "sat_scan_strided",
                 2.0 * (double)(outer * n * inner) * es, st);
    *launches += launch_scan(dtype, op, src, dst, outer, n, inner, L, nseg, rev, st);
  }
  if (nseg > 1) {
    void* tot = ar.take((size_t)(outer * (nseg - 1) * inner) * es);
    if (live) *launches += launch_seg_carry(dtype, op, dst, tot, outer, n, inner, L, nseg, rev, 0, st);
    // totals are stored in (possibly reversed) line order: a forward scan
    int rc = scan_view(dtype, tot, tot, outer, nseg - 1, inner, ar, st, launches, op, 0);
    if (rc) return rc;
    if (live) *launches += launch_seg_carry(dtype, op, dst, tot, outer, n, inner, L, nseg, rev, 1, st);
  }
  return EXSUM_OK;
}

// "sat" / "satc" (included.py:98-121, excluded.py:83-85) on an invertible +
// monoid: the running-sum table in workspace, then the 2^d-corner query with
// the route epilogue.  `total` (satc) comes from the caller when given.
int route_sat(const Shape& s, int dtype, const void* in, void* out, Arena& ar, int qmode,
              const void* given_total, const FastMod& fm, cudaStream_t st, int* launches) {
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  const void* table = in;
  void* S = nullptr;
  bool have_table = false;
  for (int a = 0; a < s.d; ++a) {
    if (s.ext[a] == 1) continue;  // accumulate over one element is a copy
    if (!have_table) S = ar.take((size_t)s.N * es);
    have_table = true;
    int rc = scan_view(dtype, table, S, prod(s.ext, 0, a), s.ext[a], prod(s.ext, a + 1, s.d), ar,
                       st, launches);
    if (rc) return rc;
    table = S;
  }
  const void* total = given_total;
  if (qmode == QUERY_COMPLEMENT && !total) {
    void* partials = ar.take((size_t)reduce_partials_count() * 8);
    void* t = ar.take(8);
    if (live) {
      ProfScope ps("total", (double)s.N * es, st);
      *launches += launch_total(dtype, EXSUM_ADD, in, s.N, partials, t, st);
    }
    total = t;
  }
  if (live) {
    QShape q;
    q.d = s.d;
    int64_t stride = 1;
    for (int j = s.d - 1; j >= 0; --j) {
      q.ext[j] = s.ext[j];
      q.k[j] = s.k[j];
      q.str[j] = stride;
      stride *= s.ext[j];
    }
    ProfScope ps("sat_query", 2.0 * (double)s.N * es, st);
    *launches += launch_sat_query(dtype, table, out, q, s.N, total, qmode, fm, st);
  }
  return EXSUM_OK;
}

// "corners" / "corners-spine" (excluded.py:191-292; 2-D and 3-D): for every
// pattern in sorted order, a copy of A accumulated along axes 0..d-1 (P:
// forward, S: reversed; sequential per line like numpy) and its contribution
// combined into out.  The reference's two variants differ only in how many
// scanned copies they keep (buffers / cache depth); they scan the same
// tensors and accumulate in the same order, so one device route serves both
// (its workspace is one scanned copy, the leaf-buffered form with c = 1).
int route_corners(const Shape& s, int dtype, int op, const void* in, void* out, Arena& ar,
                  cudaStream_t st, int* launches) {
  // CORNER_RULES (excluded.py:45-62) in sorted pattern order, one bit per
  // axis (bit a set: the threshold is the far face x_a + k_a)
  static const int kFar2[4] = {0b01, 0b11, 0b00, 0b10};                    // PP PS SP SS
  static const int kFar3[8] = {0b101, 0b111, 0b001, 0b011, 0b100, 0b110, 0b000, 0b010};
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  const int d = s.d;
  void* sc = ar.take((size_t)s.N * es);
  CornerSpec cs;
  cs.d = d;
  int64_t stride = 1;
  for (int a = d - 1; a >= 0; --a) {
    cs.ext[a] = s.ext[a];
    cs.k[a] = s.k[a];
    cs.str[a] = stride;
    stride *= s.ext[a];
  }
  for (int p = 0; p < (1 << d); ++p) {
    const int far_msb = d == 2 ? kFar2[p] : kFar3[p];  // bit (d-1-a) <-> axis a
    cs.suffix = 0;
    cs.far = 0;
    for (int a = 0; a < d; ++a) {
      if ((p >> (d - 1 - a)) & 1) cs.suffix |= 1 << a;
      if ((far_msb >> (d - 1 - a)) & 1) cs.far |= 1 << a;
    }
    const void* cur = in;
    for (int a = 0; a < d; ++a) {
      int rc = scan_view(dtype, cur, sc, prod(s.ext, 0, a), s.ext[a], prod(s.ext, a + 1, d), ar,
                         st, launches, op, (cs.suffix >> a) & 1);
      if (rc) return rc;
      cur = sc;
    }
    if (live) {
      ProfScope ps("corner_apply", (p == 0 ? 2.0 : 3.0) * (double)s.N * es, st);
      *launches += launch_corner_apply(dtype, op, sc, out, cs, s.N, p == 0, st);
    }
  }
  return EXSUM_OK;
}

// mod-add:<m> (monoid.py:235-286).  Every route of the reference yields
// (the exact integer fold) mod m, with one exception: elements that no
// combine of bdbs touched keep their raw input value (windowed_sum_axis
// leaves the last element of a line alone for 1 < k < n and the whole line
// for k == 1; an accumulate, k >= n, reduces every element).  So: canonical
// residues (int64 sums of N < 2^32 residues below 2^31 cannot overflow),
// the exact int64 + route, then the mod-m epilogue, and the raw slice copied
// back for bdbs / bdbsc.  The bdbsc / satc total is the wrapping int64 sum of
// the raw input, reduced mod m (ModAddOps.fold: int(arr.sum()) % m).
int route_modadd(int route, const Shape& s, int64_t modulus, const void* in, void* out, Arena& ar,
                 cudaStream_t st, int* launches) {
  const bool live = ar.base != nullptr;
  const FastMod fm = make_fastmod(modulus);
  const size_t bytes = (size_t)s.N * 8;
  void* total = nullptr;
  if (route == EXSUM_ROUTE_BDBSC || route == EXSUM_ROUTE_SATC) {
    void* partials = ar.take((size_t)reduce_partials_count() * 8);
    total = ar.take(8);
    if (live) {
      ProfScope ps("total", (double)bytes, st);
      *launches += launch_total(EXSUM_I64, EXSUM_ADD, in, s.N, partials, total, st);
    }
  }
  bool all_k1 = true, accumulated = false;
  SliceSpec sp;
  sp.d = s.d;
  int64_t slice = 1;
  for (int j = 0; j < s.d; ++j) {
    sp.ext[j] = s.ext[j];
    sp.fixed[j] = s.k[j] > 1;
    if (s.k[j] > 1) all_k1 = false;
    if (s.k[j] > 1 && s.k[j] >= s.ext[j]) accumulated = true;
    if (s.k[j] == 1) slice *= s.ext[j];
  }
  const bool raw_route = route == EXSUM_ROUTE_BDBS || route == EXSUM_ROUTE_BDBSC;
  if (raw_route && all_k1) {  // bdbs is a plain copy: nothing is reduced
    if (live) {
      ProfScope ps(route == EXSUM_ROUTE_BDBS ? "copy" : "mod_map", 2.0 * (double)bytes, st);
      if (route == EXSUM_ROUTE_BDBS) {
        cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice, st);
      } else {
        *launches += launch_mod_map(in, out, s.N, 1, fm, total, st);
      }
    }
    return EXSUM_OK;
  }
  void* canon = ar.take(bytes);
  if (live) {
    ProfScope ps("mod_map", 2.0 * (double)bytes, st);
    *launches += launch_mod_map(in, canon, s.N, 0, fm, nullptr, st);
  }
  int rc = EXSUM_OK;
  switch (route) {
    case EXSUM_ROUTE_SAT:
    case EXSUM_ROUTE_SATC:
      return route_sat(s, EXSUM_I64, canon, out, ar,
                       route == EXSUM_ROUTE_SAT ? QUERY_MOD : QUERY_MOD_COMPLEMENT, total, fm, st,
                       launches);
    case EXSUM_ROUTE_BOX_COMPLEMENT:
      rc = route_box_complement(s, EXSUM_I64, EXSUM_ADD, canon, out, ar, st, launches);
      break;
    case EXSUM_ROUTE_CORNERS:
    case EXSUM_ROUTE_CORNERS_SPINE:
      rc = route_corners(s, EXSUM_I64, EXSUM_ADD, canon, out, ar, st, launches);
      break;
    default:
      rc = route_bdbs(s, EXSUM_I64, EXSUM_ADD, canon, out, ar, false, st, launches);
      break;
  }
  if (rc) return rc;
  if (!live) return EXSUM_OK;
  // bdbs: reduce, then put the untouched raw elements back; bdbsc: the
  // complement reads them raw (np.subtract(total, dst) then np.remainder)
  auto raw_slice = [&]() {
    if (raw_route && !accumulated) {
      ProfScope ps("copy_slice", 2.0 * (double)slice * 8, st);
      *launches += launch_copy_slice(in, out, sp, slice, st);
    }
  };
  if (route == EXSUM_ROUTE_BDBSC) raw_slice();
  {
    ProfScope ps("mod_map", 2.0 * (double)bytes, st);
    *launches += launch_mod_map(out, out, s.N, route == EXSUM_ROUTE_BDBSC ? 1 : 0, fm, total, st);
  }
  if (route == EXSUM_ROUTE_BDBS) raw_slice();
  return EXSUM_OK;
}

int dispatch(int route, const Shape& s, int dtype, int op, int64_t modulus, const void* in,
             void* out, Arena& ar, cudaStream_t st, int* launches) {
  if (op == EXSUM_MODADD) return route_modadd(route, s, modulus, in, out, ar, st, launches);
  const FastMod fm = make_fastmod(2);
  switch (route) {
    case EXSUM_ROUTE_BDBS:
      return route_bdbs(s, dtype, op, in, out, ar, false, st, launches);
    case EXSUM_ROUTE_BDBSC:
      return route_bdbs(s, dtype, op, in, out, ar, true, st, launches);
    case EXSUM_ROUTE_BOX_COMPLEMENT:
      return route_box_complement(s, dtype, op, in, out, ar, st, launches);
    case EXSUM_ROUTE_SAT:
      return route_sat(s, dtype, in, out, ar, QUERY_PLAIN, nullptr, fm, st, launches);
    case EXSUM_ROUTE_SATC:
      return route_sat(s, dtype, in, out, ar, QUERY_COMPLEMENT, nullptr, fm, st, launches);
    case EXSUM_ROUTE_CORNERS:
    case EXSUM_ROUTE_CORNERS_SPINE:
      return route_corners(s, dtype, op, in, out, ar, st, launches);
  }
  return fail(EXSUM_ECONFIG, "unknown route");
}

int validate(int route, int dtype, int op, int64_t modulus, int d, const int64_t* ext,
             const int64_t* box, Shape* s) {
  int rc = check_types(dtype, op, modulus);
  if (rc) return rc;
  if (route < 0 || route > EXSUM_ROUTE_CORNERS_SPINE) return fail(EXSUM_ECONFIG, "unknown route");
  // _corner_rules (excluded.py:191-197): rule tables exist for 2-D and 3-D only
  if ((route == EXSUM_ROUTE_CORNERS || route == EXSUM_ROUTE_CORNERS_SPINE) && d != 2 && d != 3)
    return fail(EXSUM_ECONFIG, "corner decomposition is only defined for 2-D and 3-D tensors, got " +
                                   std::to_string(d) + "-D");
  // bench.check_algorithm_config (bench.py:88-100): bdbsc, sat and satc need
  // an inverse (bench.py:61-69, needs_inverse)
  if (op == EXSUM_MAX &&
      (route == EXSUM_ROUTE_BDBSC || route == EXSUM_ROUTE_SAT || route == EXSUM_ROUTE_SATC)) {
    const char* name = route == EXSUM_ROUTE_BDBSC ? "bdbsc" : route == EXSUM_ROUTE_SAT ? "sat" : "satc";
    return fail(EXSUM_ECONFIG, std::string("algorithm '") + name +
                                   "' requires an invertible monoid, but 'max-i64' has no inverse");
  }
  return normalize(d, ext, box, s);
}

thread_local int g_last_launches = 0;
thread_local long long g_total_launches = 0;

int run_device(int route, const void* in, void* out, int dtype, int op, int64_t modulus, int d,
               const int64_t* ext, const int64_t* box, void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  Shape s;
  int rc = validate(route, dtype, op, modulus, d, ext, box, &s);
  if (rc) return rc;
  if (!in || !out) return fail(EXSUM_EUSAGE, "null array pointer");
  if (in == out) return fail(EXSUM_EUSAGE, "out must not alias in");
  Arena sizing(nullptr);
  int launches = 0;
  rc = dispatch(route, s, dtype, op, modulus, in, out, sizing, (cudaStream_t)stream, &launches);
  if (rc) return rc;
  if (sizing.off > 0 && (ws == nullptr || ws_bytes < sizing.off))
    return fail(EXSUM_EUSAGE, "workspace too small (see exsum_workspace_bytes)");
  Arena ar(ws);
  launches = 0;
  rc = dispatch(route, s, dtype, op, modulus, in, out, ar, (cudaStream_t)stream, &launches);
  if (rc) return rc;
  g_last_launches = launches;
  g_total_launches += launches;
  return cuda_check("kernel launch");
}


// ------------------------------------------------ CUDA-graph replay --
// A device call repeated with the same arguments (route, shape, box, the
// same in / out / workspace pointers -- a training or serving loop) is
// captured once into a CUDA graph on a private stream and replayed with one
// cudaGraphLaunch on the caller's stream: no per-call planning on the host
// and no host launch gaps between the route's short kernels (C2: 6 launches,
// 3-10 us each besides the two full passes).  First sighting of a key runs
// directly; the second captures; later ones replay.  Anything the capture
// cannot take (an error, the profiler on, EXSUM_GRAPH=0) runs directly.
namespace {
struct GraphEntry {
  int route = 0, dtype = 0, op = 0, d = 0, dev = -1;
  int64_t modulus = 0;
  int64_t ext[EXSUM_MAX_DIMS] = {}, box[EXSUM_MAX_DIMS] = {};
  const void* in = nullptr;
  void* out = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  uint64_t envh = 0;  // the EXSUM_* knobs the plan read
  int seen = 0;
  bool bad = false;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
  uint64_t used = 0;
};
struct GraphCache {
  std::mutex mu;
  std::vector<GraphEntry> e;
  std::vector<std::pair<int, cudaStream_t>> cap;  // capture stream per device
  uint64_t tick = 0;
};
GraphCache& graph_cache() {
  static GraphCache c;
  return c;
}
bool graphs_on() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("EXSUM_GRAPH");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
constexpr size_t kGraphCap = 32;
// hash of the EXSUM_* environment: the planners read several knobs per call,
// so a graph is only replayed under the settings it was captured with
uint64_t exsum_env_hash() {
  uint64_t h = 1469598103934665603ull;
  for (char** e = environ; e && *e; ++e) {
    if (strncmp(*e, "EXSUM_", 6) != 0) continue;
    for (const char* p = *e; *p; ++p) h = (h ^ (unsigned char)*p) * 1099511628211ull;
    h = (h ^ 0xff) * 1099511628211ull;
  }
  return h;
}
}  // namespace

int run_device_graph(int route, const void* in, void* out, int dtype, int op, int64_t modulus,
                     int d, const int64_t* ext, const int64_t* box, void* ws, size_t ws_bytes,
                     void* stream) {
  if (!graphs_on() || g_prof.on || d < 1 || d > EXSUM_MAX_DIMS || !ext || !box || !in || !out ||
      in == out)
    return run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
  {  // argument errors report exactly as the direct path (before any CUDA call)
    Shape sh;
    if (validate(route, dtype, op, modulus, d, ext, box, &sh) != EXSUM_OK)
      return run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  const uint64_t envh = exsum_env_hash();
  GraphCache& c = graph_cache();
  std::unique_lock<std::mutex> lock(c.mu);
  GraphEntry* hit = nullptr;
  for (auto& g : c.e) {
    if (g.route != route || g.dtype != dtype || g.op != op || g.d != d || g.dev != dev ||
        g.modulus != modulus || g.in != in || g.out != out || g.ws != ws || g.ws_bytes != ws_bytes ||
        g.envh != envh)
      continue;
    bool same = true;
    for (int i = 0; i < d; ++i) same = same && g.ext[i] == ext[i] && g.box[i] == box[i];
    if (same) {
      hit = &g;
      break;
    }
  }
  if (!hit) {
    if (c.e.size() >= kGraphCap) {  // evict the least recently used
      size_t lru = 0;
      for (size_t i = 1; i < c.e.size(); ++i)
        if (c.e[i].used < c.e[lru].used) lru = i;
      if (c.e[lru].exec) cudaGraphExecDestroy(c.e[lru].exec);
      c.e.erase(c.e.begin() + (long)lru);
    }
    GraphEntry g;
    g.route = route, g.dtype = dtype, g.op = op, g.d = d, g.dev = dev, g.modulus = modulus;
    for (int i = 0; i < d; ++i) g.ext[i] = ext[i], g.box[i] = box[i];
    g.in = in, g.out = out, g.ws = ws, g.ws_bytes = ws_bytes;
    g.envh = envh;
    g.seen = 1;
    g.used = ++c.tick;
    c.e.push_back(g);
    lock.unlock();
    return run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
  }
  hit->used = ++c.tick;
  if (hit->bad) {
    lock.unlock();
    return run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
  }
  if (!hit->exec) {
    // second sighting: capture on this device's private stream
    cudaStream_t cs = nullptr;
    for (auto& p : c.cap)
      if (p.first == dev) cs = p.second;
    if (!cs) {
      if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        hit->bad = true;
        lock.unlock();
        return run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
      }
      c.cap.push_back({dev, cs});
    }
    cudaGraph_t graph = nullptr;
    int rc = EXSUM_OK;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      rc = run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, (void*)cs);
      const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
      if (ce != cudaSuccess) rc = rc ? rc : EXSUM_ECUDA;
    } else {
      rc = EXSUM_ECUDA;
    }
    cudaGraphExec_t exec = nullptr;
    if (rc == EXSUM_OK && graph && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) exec = nullptr;
    if (graph) cudaGraphDestroy(graph);
    if (rc != EXSUM_OK || !exec) {
      cudaGetLastError();  // clear a capture error; the direct call reports its own
      hit->bad = true;
      lock.unlock();
      return run_device(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
    }
    hit->exec = exec;
    hit->launches = g_last_launches;
    g_total_launches -= g_last_launches;  // captured, not launched
  }
  const cudaGraphExec_t exec = hit->exec;
  const int launches = hit->launches;
  g_err.clear();
  // launched under the cache lock (the launch is asynchronous and cheap): an
  // eviction or exsum_release_cache on another thread cannot destroy `exec`
  // between the lookup and the launch
  const cudaError_t le = cudaGraphLaunch(exec, (cudaStream_t)stream);
  lock.unlock();
  if (le != cudaSuccess) return cuda_check("cudaGraphLaunch");
  g_last_launches = launches;
  g_total_launches += launches;
  return EXSUM_OK;
}

void release_graphs() {
  GraphCache& c = graph_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  for (auto& g : c.e)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  c.e.clear();
}

// ----------------------------------------------------- shard stages (8e) --
// Axis-0 sharding (paper_2106_00124_b200/sharded.py): a rank owns planes
// [x_s, x_e) of axis 0 and receives the next rank's first k0-1 planes as a
// halo.  Stage 1 runs the axis-0 windowed pass over own+halo planes producing
// only the own planes (optionally folding the raw own planes into R or the
// local total); stage 2 finishes BDBS/BDBSC (remaining axes, global total) or
// box-complement (remaining W passes + row round with the tail slice).

int stage_axis0(const Shape& s, int64_t n_out, int64_t k0, int dtype, int op, const void* in,
                void* out, int extra_kind, void* extra_out, Arena& ar, cudaStream_t st,
                int* launches) {
  const size_t es = dtype_size(dtype);
  const bool live = ar.base != nullptr;
  const int d = s.d;
  const int64_t n_in = s.ext[0];
  const int64_t inner = s.N / n_in;
  const int64_t N_out = n_out * inner;
  const int64_t row_len = s.ext[d - 1];
  const int64_t rows_out = N_out / row_len;
  const int64_t k = k0 < n_in ? k0 : n_in;
  void* partials = ar.take((size_t)reduce_partials_count() * 8);
  void* rowpart = extra_kind == 1 ? ar.take((size_t)(N_out / 32 + 1) * es) : nullptr;
  void* tmp = (k > 1 && n_out != n_in) ? ar.take((size_t)s.N * es) : nullptr;
  if (!live) return EXSUM_OK;
  PassExtra ex;
  bool extras_done = false;
  if (k == 1) {
    cudaMemcpyAsync(out, in, (size_t)N_out * es, cudaMemcpyDeviceToDevice, st);
  } else {
    ex.kind = extra_kind;
    ex.buf = extra_kind == 1 ? rowpart : partials;
    ex.row_len = row_len;
    ex.cap = reduce_partials_count();
    ex.n_out = n_out == n_in ? -1 : n_out;
    {
      ProfScope ps("shard_axis0", (double)(n_in * inner + N_out) * es, st);
      int rc = launch_pass(dtype, op, in, out, 1, n_in, inner, k, nullptr, st, &ex);
      if (rc < 0) return fail(EXSUM_ECONFIG, "no kernel for this dtype/operator");
      *launches += rc;
    }
    if (ex.n_out >= 0 && !ex.n_out_done) {
      // the pass kernel for this shape cannot stop at n_out: full-length pass
      // into a temporary, then keep the own planes
      PassExtra plain;
      int rc = launch_pass(dtype, op, in, tmp, 1, n_in, inner, k, nullptr, st, &plain);
      if (rc < 0) return fail(EXSUM_ECONFIG, "no kernel for this dtype/operator");
      *launches += rc;
      cudaMemcpyAsync(out, tmp, (size_t)N_out * es, cudaMemcpyDeviceToDevice, st);
    } else {
      extras_done = ex.done != 0;
    }
  }
  if (extra_kind == 1) {
    if (extras_done)
      *launches += launch_rowpart_final(dtype, op, rowpart, extra_out, rows_out, ex.ppr, st);
    else
      *launches += launch_row_reduce(dtype, op, in, extra_out, rows_out, row_len, st);
  } else if (extra_kind == 2) {
    if (extras_done)
      *launches += launch_total_final(dtype, op, partials, ex.ppr, extra_out, st);
    else
      *launches += launch_total(dtype, op, in, N_out, partials, extra_out, st);
  }
  return EXSUM_OK;
}

int stage_bc_finish(const Shape& s, int dtype, int op, const void* in, void* out, const void* T,
                    Arena& ar, cudaStream_t st, int* launches) {
  const int d = s.d;
  PassPlan p = plan_passes(s, d - 1);
  PassPlan head;  // axis 0 was done by stage 1
  for (int i = 0; i < p.count; ++i)
    if (p.axes[i] != 0) head.axes[head.count++] = p.axes[i];
  const bool fused = head.count > 0 && head.axes[head.count - 1] == d - 2 &&
                     fused_pair_ok(dtype, op, s.ext[d - 1], s.k[d - 2], s.k[d - 1], ROW_EXCL) &&
                     aligned16(out) && (head.count > 1 || aligned16(in));
  if (fused) head.count -= 1;
  return bc_finish(s, dtype, op, in, out, T, head, fused, nullptr, no_hook, ar, st, launches);
}

// stage 0: axis-0 shard pass; 1: bdbs/bdbsc finish; 2: box-complement finish
int run_stage(int stage, int dtype, int op, int d, const int64_t* ext, const int64_t* box,
              int64_t n_out, int extra_kind, const void* in, void* out, const void* aux,
              void* extra_out, Arena& ar, cudaStream_t st, int* launches) {
  Shape s;
  int rc = check_types(dtype, op);
  if (rc) return rc;
  rc = normalize(d, ext, box, &s);
  if (rc) return rc;
  if (stage == 0) {
    if (n_out < 1 || n_out > s.ext[0]) return fail(EXSUM_EUSAGE, "n_out must be in [1, ext[0]]");
    if (n_out != s.ext[0] && box[0] > 1 && n_out % box[0] != 0)
      return fail(EXSUM_EUSAGE, "a shard's own planes must be a multiple of the axis-0 window");
    if (extra_kind < 0 || extra_kind > 2) return fail(EXSUM_EUSAGE, "extra_kind must be 0, 1 or 2");
    if (extra_kind == 2 && op == EXSUM_MAX) return fail(EXSUM_ECONFIG, "no total for max-i64 (bdbsc needs an inverse)");
    return stage_axis0(s, n_out, box[0], dtype, op, in, out, extra_kind, extra_out, ar, st, launches);
  }
  s.k[0] = 1;
  if (stage == 1) return route_bdbs(s, dtype, op, in, out, ar, aux != nullptr, st, launches, aux);
  if (stage == 2) {
    if (d < 2) return fail(EXSUM_ECONFIG, "sharded box-complement needs d >= 2");
    s.k[0] = box[0] < ext[0] ? box[0] : ext[0];
    return stage_bc_finish(s, dtype, op, in, out, aux, ar, st, launches);
  }
  return fail(EXSUM_EUSAGE, "unknown stage");
}

int run_stage_device(int stage, int dtype, int op, int d, const int64_t* ext, const int64_t* box,
                     int64_t n_out, int extra_kind, const void* in, void* out, const void* aux,
                     void* extra_out, void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (!in || !out || in == out) return fail(EXSUM_EUSAGE, "need distinct in/out");
  Arena sizing(nullptr);
  int launches = 0;
  int rc = run_stage(stage, dtype, op, d, ext, box, n_out, extra_kind, in, out, aux, extra_out,
                     sizing, (cudaStream_t)stream, &launches);
  if (rc) return rc;
  if (sizing.off > 0 && (ws == nullptr || ws_bytes < sizing.off))
    return fail(EXSUM_EUSAGE, "workspace too small (see exsum_shard_workspace_bytes)");
  Arena ar(ws);
  launches = 0;
  rc = run_stage(stage, dtype, op, d, ext, box, n_out, extra_kind, in, out, aux, extra_out, ar,
                 (cudaStream_t)stream, &launches);
  if (rc) return rc;
  g_last_launches = launches;
  g_total_launches += launches;
  return cuda_check("kernel launch");
}

// ----------------------------------------------------- host buffer cache --
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return -1;
    cap = bytes;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct HostCache {
  std::mutex mu;
  std::vector<int> dev;
  std::vector<DevBuf> in, out, ws;
  std::vector<cudaStream_t> stream;
};

// exsum_route_host_batch: two device slots and three streams per device, so
// the copy engines run both directions at once (PCIe is full duplex: ~56 GB/s
// each way, ~100 GB/s together, measured on B200 boxes) while a slot computes.
struct BatchSlot {
  DevBuf in, out, ws;
  cudaEvent_t h2d = nullptr, done = nullptr, d2h = nullptr;
};
struct BatchCache {
  std::mutex mu;
  std::vector<int> dev;
  std::vector<BatchSlot> slots;  // 2 per device
  std::vector<cudaStream_t> streams;  // 3 per device: h2d, compute, d2h
};
BatchCache& batch_cache() {
  static BatchCache c;
  return c;
}

HostCache& host_cache() {
  static HostCache c;
  return c;
}

}  // namespace

extern "C" {

int exsum_abi_version(void) { return EXSUM_ABI_VERSION; }

const char* exsum_last_error(void) { return g_err.c_str(); }

int exsum_last_launch_count(void) { return g_last_launches; }

long long exsum_total_launch_count(void) { return g_total_launches; }

int exsum_route_workspace_bytes(int route, int dtype, int op, int64_t modulus, int d,
                                const int64_t* ext, const int64_t* box, size_t* bytes) {
  g_err.clear();
  Shape s;
  int rc = validate(route, dtype, op, modulus, d, ext, box, &s);
  if (rc) return rc;
  Arena sizing(nullptr);
  int launches = 0;
  // the larger of the plans for 16-byte aligned arrays (every CUDA allocation)
  // and for arrays off that alignment (unfused kernels; the two differ only
  // for 2-D box-complement); run_device re-plans with the caller's pointers
  rc = dispatch(route, s, dtype, op, modulus, (const void*)256, (void*)512, sizing, nullptr,
                &launches);
  if (rc) return rc;
  Arena sizing_u(nullptr);
  rc = dispatch(route, s, dtype, op, modulus, (const void*)8, (void*)24, sizing_u, nullptr,
                &launches);
  if (rc) return rc;
  if (bytes) *bytes = sizing.off > sizing_u.off ? sizing.off : sizing_u.off;
  return EXSUM_OK;
}

int exsum_workspace_bytes(int route, int dtype, int op, int d, const int64_t* ext,
                          const int64_t* box, size_t* bytes) {
  return exsum_route_workspace_bytes(route, dtype, op, 0, d, ext, box, bytes);
}

int exsum_route(int route, const void* in, void* out, int dtype, int op, int64_t modulus, int d,
                const int64_t* ext, const int64_t* box, void* ws, size_t ws_bytes, void* stream) {
  return run_device_graph(route, in, out, dtype, op, modulus, d, ext, box, ws, ws_bytes, stream);
}

int exsum_bdbs_included(const void* in, void* out, int dtype, int op, int d, const int64_t* ext,
                        const int64_t* box, void* ws, size_t ws_bytes, void* stream) {
  return run_device_graph(EXSUM_ROUTE_BDBS, in, out, dtype, op, 0, d, ext, box, ws, ws_bytes, stream);
}

int exsum_bdbsc_excluded(const void* in, void* out, int dtype, int op, int d, const int64_t* ext,
                         const int64_t* box, void* ws, size_t ws_bytes, void* stream) {
  return run_device_graph(EXSUM_ROUTE_BDBSC, in, out, dtype, op, 0, d, ext, box, ws, ws_bytes, stream);
}

int exsum_box_complement_excluded(const void* in, void* out, int dtype, int op, int d,
                                  const int64_t* ext, const int64_t* box, void* ws,
                                  size_t ws_bytes, void* stream) {
  return run_device_graph(EXSUM_ROUTE_BOX_COMPLEMENT, in, out, dtype, op, 0, d, ext, box, ws, ws_bytes,
                    stream);
}

int exsum_windowed_pass(const void* in, void* out, int dtype, int op, int d, const int64_t* ext,
                        int axis, int64_t k, void* stream) {
  g_err.clear();
  int rc = check_types(dtype, op);
  if (rc) return rc;
  if (d < 1 || d > EXSUM_MAX_DIMS || !ext) return fail(EXSUM_EUSAGE, "bad extents");
  if (axis < 0 || axis >= d) return fail(EXSUM_EUSAGE, "axis out of range");
  if (k < 1) return fail(EXSUM_EUSAGE, "window must be >= 1");
  if (!in || !out || in == out) return fail(EXSUM_EUSAGE, "need distinct in/out");
  for (int i = 0; i < d; ++i)
    if (ext[i] < 1) return fail(EXSUM_EUSAGE, "every extent must be >= 1");
  const int64_t n = ext[axis];
  if (k > n) k = n;
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 1) {
    cudaMemcpyAsync(out, in, (size_t)prod(ext, 0, d) * dtype_size(dtype), cudaMemcpyDeviceToDevice, st);
    g_last_launches = 0;
  } else {
    rc = launch_pass(dtype, op, in, out, prod(ext, 0, axis), n, prod(ext, axis + 1, d), k, nullptr, st);
    if (rc < 0) return fail(EXSUM_ECONFIG, "no kernel for this dtype/operator");
    g_last_launches = rc;
    g_total_launches += rc;
  }
  return cuda_check("kernel launch");
}

// BDBS on host buffers, pipelined over axis-0 chunks: output planes depend only
// on input planes [x0, x0 + k0 - 1], so chunk j (a multiple of k0 planes) runs
// the axis-0 shard stage (its halo is chunk j+1's first k0-1 planes, already in
// the device copy) and the finish stage while chunk j+1 is copied in and chunk
// j-1 is copied out -- the copy engines run both directions at once.  Block-
// aligned chunks keep the reference's association: bit-identical to one call.
static int bdbs_host_pipelined(const Shape& s, const int64_t* box, const void* h_in, void* h_out,
                        int dtype, int op) {
  const size_t es = dtype_size(dtype);
  const int d = s.d;
  const int64_t n0 = s.ext[0], k0 = s.k[0];
  const int64_t plane = s.N / n0;
  int64_t P = (n0 + 15) / 16;  // ~16 chunks: the unoverlapped first H2D / last D2H is 1/16
  P = (P + k0 - 1) / k0 * k0;
  const int64_t nch = (n0 + P - 1) / P;
  int64_t ext_c[EXSUM_MAX_DIMS];
  for (int i = 0; i < d; ++i) ext_c[i] = s.ext[i];
  // workspace: the axis-0 stage output (P planes) + the larger stage workspace
  size_t ws0 = 0, ws1 = 0;
  {
    ext_c[0] = P + (k0 - 1 < n0 - P ? k0 - 1 : (n0 - P > 0 ? n0 - P : 0));
    Arena a0(nullptr);
    int l = 0;
    int rc = run_stage(0, dtype, op, d, ext_c, box, P, 0, (const void*)256, (void*)512, nullptr,
                       nullptr, a0, nullptr, &l);
    if (rc) return rc;
    ws0 = a0.off;
    ext_c[0] = P;
    Arena a1(nullptr);
    rc = run_stage(1, dtype, op, d, ext_c, box, 0, 0, (const void*)256, (void*)512, nullptr,
                   nullptr, a1, nullptr, &l);
    if (rc) return rc;
    ws1 = a1.off;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  BatchCache& c = batch_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  size_t di = 0;
  while (di < c.dev.size() && c.dev[di] != dev) ++di;
  if (di == c.dev.size()) {
    c.dev.push_back(dev);
    for (int k = 0; k < 2; ++k) {
      BatchSlot b;
      if (cudaEventCreateWithFlags(&b.h2d, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&b.d2h, cudaEventDisableTiming) != cudaSuccess)
        return cuda_check("cudaEventCreate");
      c.slots.push_back(b);
    }
    for (int k = 0; k < 3; ++k) {
      cudaStream_t st;
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return cuda_check("cudaStreamCreate");
      c.streams.push_back(st);
    }
  }
  // buffers: slot 0 holds the whole input and output; slot 1's `in` the stage
  // output, its `ws` the stage workspace
  BatchSlot* slot = &c.slots[2 * di];
  const size_t bytes = (size_t)s.N * es;
  const size_t ybytes = (size_t)(P * plane) * es;
  const size_t wsb = (ws0 > ws1 ? ws0 : ws1) > 0 ? (ws0 > ws1 ? ws0 : ws1) : 256;
  if (slot[0].in.reserve(bytes) || slot[0].out.reserve(bytes) || slot[1].in.reserve(ybytes) ||
      slot[1].ws.reserve(wsb))
    return fail(EXSUM_ECUDA, "cudaMalloc failed for the pipelined host path");
  cudaStream_t s_in = c.streams[3 * di], s_run = c.streams[3 * di + 1], s_out = c.streams[3 * di + 2];
  std::vector<cudaEvent_t> ev(3 * nch);
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return cuda_check("cudaEventCreate");
  char* din = (char*)slot[0].in.p;
  char* dout = (char*)slot[0].out.p;
  for (int64_t j = 0; j < nch; ++j) {
    const int64_t a = j * P, b = a + P < n0 ? a + P : n0;
    cudaMemcpyAsync(din + a * plane * es, (const char*)h_in + a * plane * es,
                    (size_t)((b - a) * plane) * es, cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(ev[3 * j], s_in);
  }
  int rc = EXSUM_OK;
  for (int64_t j = 0; j < nch && rc == EXSUM_OK; ++j) {
    const int64_t a = j * P, b = a + P < n0 ? a + P : n0;
    const int64_t own = b - a;
    const int64_t halo = k0 - 1 < n0 - b ? k0 - 1 : n0 - b;
    cudaStreamWaitEvent(s_run, ev[3 * j], 0);
    if (halo > 0) cudaStreamWaitEvent(s_run, ev[3 * (j + 1)], 0);
    if (j >= 1) cudaStreamWaitEvent(s_run, ev[3 * (j - 1) + 1], 0);  // y / ws reuse (same stream)
    ext_c[0] = own + halo;
    int l = 0;
    if (k0 > 1) {
      Arena ar(slot[1].ws.p);
      rc = run_stage(0, dtype, op, d, ext_c, box, own, 0, din + a * plane * es, slot[1].in.p,
                     nullptr, nullptr, ar, s_run, &l);
      if (rc) break;
    }
    ext_c[0] = own;
    Arena ar1(slot[1].ws.p);
    rc = run_stage(1, dtype, op, d, ext_c, box, 0, 0, k0 > 1 ? slot[1].in.p : din + a * plane * es,
                   dout + a * plane * es, nullptr, nullptr, ar1, s_run, &l);
    g_total_launches += l;
    cudaEventRecord(ev[3 * j + 1], s_run);
    cudaStreamWaitEvent(s_out, ev[3 * j + 1], 0);
    cudaMemcpyAsync((char*)h_out + a * plane * es, dout + a * plane * es,
                    (size_t)(own * plane) * es, cudaMemcpyDeviceToHost, s_out);
  }
  cudaError_t e1 = cudaStreamSynchronize(s_in);
  cudaError_t e2 = cudaStreamSynchronize(s_run);
  cudaError_t e3 = cudaStreamSynchronize(s_out);
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc) return rc;
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
    return cuda_check("pipelined host path");
  return cuda_check("pipelined host path");
}

int exsum_route_host(int route, const void* h_in, void* h_out, int dtype, int op, int64_t modulus,
                     int d, const int64_t* ext, const int64_t* box) {
  g_err.clear();
  Shape s;
  int rc = validate(route, dtype, op, modulus, d, ext, box, &s);
  if (rc) return rc;
  if (!h_in || !h_out) return fail(EXSUM_EUSAGE, "null host pointer");
  if (route == EXSUM_ROUTE_BDBS && op != EXSUM_MODADD && d >= 2 &&
      (size_t)s.N * dtype_size(dtype) >= ((size_t)64 << 20) && s.ext[0] >= 4 * s.k[0] &&
      s.ext[0] >= 16) {
    int64_t kb[EXSUM_MAX_DIMS];
    for (int i = 0; i < d; ++i) kb[i] = s.k[i];
    return bdbs_host_pipelined(s, kb, h_in, h_out, dtype, op);
  }
  size_t ws_bytes = 0;
  rc = exsum_route_workspace_bytes(route, dtype, op, modulus, d, ext, box, &ws_bytes);
  if (rc) return rc;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  HostCache& c = host_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  size_t slot = 0;
  while (slot < c.dev.size() && c.dev[slot] != dev) ++slot;
  if (slot == c.dev.size()) {
    c.dev.push_back(dev);
    c.in.emplace_back();
    c.out.emplace_back();
    c.ws.emplace_back();
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_check("cudaStreamCreate");
    c.stream.push_back(st);
  }
  const size_t bytes = (size_t)s.N * dtype_size(dtype);
  if (c.in[slot].reserve(bytes) || c.out[slot].reserve(bytes) ||
      c.ws[slot].reserve(ws_bytes > 0 ? ws_bytes : 256))
    return fail(EXSUM_ECUDA, "cudaMalloc failed for host-path buffers");
  cudaStream_t st = c.stream[slot];
  // every exit below drains the stream first: no copy into or out of the
  // caller's buffers may still be in flight when the call returns
  if (cudaMemcpyAsync(c.in[slot].p, h_in, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    rc = cuda_check("cudaMemcpyAsync H2D");
  } else {
    rc = run_device(route, c.in[slot].p, c.out[slot].p, dtype, op, modulus, d, ext, box,
                    c.ws[slot].p, c.ws[slot].cap, st);
    if (!rc && cudaMemcpyAsync(h_out, c.out[slot].p, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = cuda_check("cudaMemcpyAsync D2H");
  }
  const cudaError_t se = cudaStreamSynchronize(st);
  if (rc) return rc;
  if (se != cudaSuccess) return cuda_check("cudaStreamSynchronize");
  return cuda_check("host path");
}

int exsum_route_host_batch(int route, int count, const void* const* h_in, void* const* h_out,
                           int dtype, int op, int64_t modulus, int d, const int64_t* ext,
                           const int64_t* box) {
  g_err.clear();
  Shape s;
  int rc = validate(route, dtype, op, modulus, d, ext, box, &s);
  if (rc) return rc;
  if (count < 0 || (count > 0 && (!h_in || !h_out))) return fail(EXSUM_EUSAGE, "bad batch arrays");
  for (int i = 0; i < count; ++i)
    if (!h_in[i] || !h_out[i]) return fail(EXSUM_EUSAGE, "null host pointer in batch");
  if (count == 0) return EXSUM_OK;
  size_t ws_bytes = 0;
  rc = exsum_route_workspace_bytes(route, dtype, op, modulus, d, ext, box, &ws_bytes);
  if (rc) return rc;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  BatchCache& c = batch_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  size_t di = 0;
  while (di < c.dev.size() && c.dev[di] != dev) ++di;
  if (di == c.dev.size()) {
    c.dev.push_back(dev);
    for (int k = 0; k < 2; ++k) {
      BatchSlot b;
      if (cudaEventCreateWithFlags(&b.h2d, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&b.d2h, cudaEventDisableTiming) != cudaSuccess)
        return cuda_check("cudaEventCreate");
      c.slots.push_back(b);
    }
    for (int k = 0; k < 3; ++k) {
      cudaStream_t st;
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return cuda_check("cudaStreamCreate");
      c.streams.push_back(st);
    }
  }
  BatchSlot* slot = &c.slots[2 * di];
  cudaStream_t s_in = c.streams[3 * di], s_run = c.streams[3 * di + 1], s_out = c.streams[3 * di + 2];
  const size_t bytes = (size_t)s.N * dtype_size(dtype);
  const int nslots = count > 1 ? 2 : 1;
  for (int k = 0; k < nslots; ++k)
    if (slot[k].in.reserve(bytes) || slot[k].out.reserve(bytes) ||
        slot[k].ws.reserve(ws_bytes > 0 ? ws_bytes : 256))
      return fail(EXSUM_ECUDA, "cudaMalloc failed for batch buffers");
  // on any failure: stop issuing, then drain all three streams before
  // returning, so no copy into or out of the caller's buffers is left in flight
  auto step = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && !rc) rc = cuda_check(what);
    return rc == 0;
  };
  for (int i = 0; i < count && !rc; ++i) {
    BatchSlot& b = slot[i % nslots];
    if (i >= nslots && !step(cudaStreamWaitEvent(s_in, b.done, 0), "cudaStreamWaitEvent"))
      break;  // compute of i-2 released `in`
    if (!step(cudaMemcpyAsync(b.in.p, h_in[i], bytes, cudaMemcpyHostToDevice, s_in), "cudaMemcpyAsync H2D") ||
        !step(cudaEventRecord(b.h2d, s_in), "cudaEventRecord") ||
        !step(cudaStreamWaitEvent(s_run, b.h2d, 0), "cudaStreamWaitEvent"))
      break;
    if (i >= nslots && !step(cudaStreamWaitEvent(s_run, b.d2h, 0), "cudaStreamWaitEvent"))
      break;  // D2H of i-2 released `out`
    rc = run_device(route, b.in.p, b.out.p, dtype, op, modulus, d, ext, box, b.ws.p, b.ws.cap,
                    s_run);
    if (rc) break;
    if (!step(cudaEventRecord(b.done, s_run), "cudaEventRecord") ||
        !step(cudaStreamWaitEvent(s_out, b.done, 0), "cudaStreamWaitEvent") ||
        !step(cudaMemcpyAsync(h_out[i], b.out.p, bytes, cudaMemcpyDeviceToHost, s_out), "cudaMemcpyAsync D2H") ||
        !step(cudaEventRecord(b.d2h, s_out), "cudaEventRecord"))
      break;
  }
  cudaError_t se = cudaSuccess;
  for (cudaStream_t q : {s_in, s_run, s_out}) {
    const cudaError_t e = cudaStreamSynchronize(q);
    if (se == cudaSuccess) se = e;
  }
  if (rc) return rc;
  if (se != cudaSuccess) return cuda_check("cudaStreamSynchronize");
  return cuda_check("host batch");
}

int exsum_run_host(int route, const void* h_in, void* h_out, int dtype, int op, int d,
                   const int64_t* ext, const int64_t* box) {
  return exsum_route_host(route, h_in, h_out, dtype, op, 0, d, ext, box);
}

// ------------------------------------------------------- building blocks --

int exsum_scan_workspace_bytes(int dtype, int op, int64_t modulus, int d, const int64_t* ext,
                               int axis, size_t* bytes) {
  g_err.clear();
  int rc = check_types(dtype, op, op == EXSUM_MODADD ? modulus : 0);
  if (rc) return rc;
  if (d < 1 || d > EXSUM_MAX_DIMS || !ext) return fail(EXSUM_EUSAGE, "bad extents");
  if (axis < 0 || axis >= d) return fail(EXSUM_EUSAGE, "axis out of range");
  for (int i = 0; i < d; ++i)
    if (ext[i] < 1) return fail(EXSUM_EUSAGE, "every extent must be >= 1");
  Arena sizing(nullptr);
  int launches = 0;
  rc = scan_view(dtype, (const void*)1, (void*)2, prod(ext, 0, axis), ext[axis],
                 prod(ext, axis + 1, d), sizing, nullptr, &launches,
                 op == EXSUM_MAX ? EXSUM_MAX : EXSUM_ADD, 0);
  if (rc) return rc;
  if (bytes) *bytes = sizing.off;
  return EXSUM_OK;
}

int exsum_scan_axis(const void* in, void* out, int dtype, int op, int64_t modulus, int d,
                    const int64_t* ext, int axis, int reverse, void* ws, size_t ws_bytes,
                    void* stream) {
  size_t need = 0;
  int rc = exsum_scan_workspace_bytes(dtype, op, modulus, d, ext, axis, &need);
  if (rc) return rc;
  if (!in || !out) return fail(EXSUM_EUSAGE, "null array pointer");
  if (need > 0 && (ws == nullptr || ws_bytes < need))
    return fail(EXSUM_EUSAGE, "workspace too small (see exsum_scan_workspace_bytes)");
  cudaStream_t st = (cudaStream_t)stream;
  Arena ar(ws);
  int launches = 0;
  // ModAddOps.accumulate (monoid.py:280-283): raw int64 running sum, then
  // np.remainder over the whole array
  rc = scan_view(dtype, in, out, prod(ext, 0, axis), ext[axis], prod(ext, axis + 1, d), ar, st,
                 &launches, op == EXSUM_MAX ? EXSUM_MAX : EXSUM_ADD, reverse != 0);
  if (rc) return rc;
  if (op == EXSUM_MODADD) launches += launch_mod_map(out, out, prod(ext, 0, d), 0, make_fastmod(modulus), nullptr, st);
  g_last_launches = launches;
  g_total_launches += launches;
  return cuda_check("scan");
}

int exsum_add_contribution(const void* src, void* dst, int dtype, int op, int64_t modulus, int d,
                           const int64_t* ext, int dim, int64_t offset, void* stream) {
  g_err.clear();
  int rc = check_types(dtype, op, op == EXSUM_MODADD ? modulus : 0);
  if (rc) return rc;
  if (d < 1 || d > EXSUM_MAX_DIMS || !ext) return fail(EXSUM_EUSAGE, "bad extents");
  if (dim < 0 || dim >= d) return fail(EXSUM_EUSAGE, "dimension out of range");
  if (!src || !dst) return fail(EXSUM_EUSAGE, "null array pointer");
  for (int i = 0; i < d; ++i)
    if (ext[i] < 1) return fail(EXSUM_EUSAGE, "every extent must be >= 1");
  const int launches = launch_add_contribution(dtype, op, make_fastmod(modulus), src, dst,
                                               prod(ext, 0, dim), ext[dim], prod(ext, dim + 1, d),
                                               offset, (cudaStream_t)stream);
  if (launches < 0) return fail(EXSUM_ECONFIG, "no kernel for this dtype/operator");
  g_last_launches = launches;
  g_total_launches += launches;
  return cuda_check("add_contribution");
}

int exsum_elementwise(void* dst, const void* src, const void* scalar, int dtype, int op,
                      int64_t modulus, int kind, int64_t n, void* stream) {
  g_err.clear();
  int rc = check_types(dtype, op, op == EXSUM_MODADD ? modulus : 0);
  if (rc) return rc;
  if (kind < 0 || kind > 2) return fail(EXSUM_EUSAGE, "unknown element operation");
  if (kind > 0 && op == EXSUM_MAX)
    return fail(EXSUM_ECONFIG, "monoid 'max-i64' has no inverse");  // monoid.py:72-78
  if (n < 0 || !dst || (kind < 2 && !src) || (kind == 2 && !scalar))
    return fail(EXSUM_EUSAGE, "bad element-operation arguments");
  if (n == 0) return EXSUM_OK;
  const int launches = launch_elementwise(dtype, op, make_fastmod(modulus), dst, src, scalar, kind,
                                          n, (cudaStream_t)stream);
  if (launches < 0) return fail(EXSUM_ECONFIG, "no kernel for this dtype/operator");
  g_last_launches = launches;
  g_total_launches += launches;
  return cuda_check("elementwise");
}

size_t exsum_fold_workspace_bytes(void) { return (size_t)reduce_partials_count() * 8 + 512; }

int exsum_fold(const void* in, void* result, int dtype, int op, int64_t modulus, int64_t n,
               void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  int rc = check_types(dtype, op, op == EXSUM_MODADD ? modulus : 0);
  if (rc) return rc;
  if (n < 0 || !result || (n > 0 && !in)) return fail(EXSUM_EUSAGE, "bad fold arguments");
  if (!ws || ws_bytes < exsum_fold_workspace_bytes())
    return fail(EXSUM_EUSAGE, "workspace too small (see exsum_fold_workspace_bytes)");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = dtype_size(dtype);
  if (n == 0) {  // MonoidOps.fold of an empty array: the identity
    static const float f0 = 0.0f;
    static const double d0 = 0.0;
    static const int64_t i0 = 0, imin = (int64_t)0x8000000000000000ULL;
    const void* idv = dtype == EXSUM_F32 ? (const void*)&f0 : dtype == EXSUM_F64 ? (const void*)&d0
                      : op == EXSUM_MAX ? (const void*)&imin : (const void*)&i0;
    cudaMemcpyAsync(result, idv, es, cudaMemcpyHostToDevice, st);
    return cuda_check("fold");
  }
  char* w = (char*)ws;
  void* acc = w;  // 8 bytes, then the partials
  void* partials = w + 256;
  int launches = launch_total(dtype, op == EXSUM_MAX ? EXSUM_MAX : EXSUM_ADD, in, n, partials, acc, st);
  launches += launch_fold_result(dtype, op, make_fastmod(modulus), acc, result, st);
  g_last_launches = launches;
  g_total_launches += launches;
  return cuda_check("fold");
}

int exsum_profile_enable(int on) {
  g_prof.on = on != 0;
  g_prof.recs.clear();
  g_prof.used = 0;
  return EXSUM_OK;
}

int exsum_profile_count(void) { return (int)g_prof.recs.size(); }

int exsum_profile_get(int i, char* name, int name_len, double* bytes, float* ms) {
  if (i < 0 || i >= (int)g_prof.recs.size()) return fail(EXSUM_EUSAGE, "profile index out of range");
  const ProfRec& r = g_prof.recs[i];
  if (name && name_len > 0) {
    snprintf(name, (size_t)name_len, "%s", r.name);
  }
  if (bytes) *bytes = r.bytes;
  if (ms) {
    float v = 0.f;
    if (cudaEventElapsedTime(&v, r.a, r.b) != cudaSuccess) return cuda_check("cudaEventElapsedTime");
    *ms = v;
  }
  return EXSUM_OK;
}

int exsum_shard_workspace_bytes(int stage, int dtype, int op, int d, const int64_t* ext,
                                const int64_t* box, int64_t n_out, int extra_kind,
                                size_t* bytes) {
  g_err.clear();
  Arena sizing(nullptr);
  int launches = 0;
  int rc = run_stage(stage, dtype, op, d, ext, box, n_out, extra_kind, (const void*)256, (void*)512,
                     (const void*)3, (void*)4, sizing, nullptr, &launches);
  if (rc) return rc;
  if (bytes) *bytes = sizing.off;
  return EXSUM_OK;
}

int exsum_shard_axis0_pass(const void* in, void* out, int dtype, int op, int d,
                           const int64_t* ext_in, const int64_t* box, int64_t n_out,
                           int extra_kind, void* extra_out, void* ws, size_t ws_bytes,
                           void* stream) {
  if (extra_kind != 0 && !extra_out) return fail(EXSUM_EUSAGE, "extra_out is required");
  return run_stage_device(0, dtype, op, d, ext_in, box, n_out, extra_kind, in, out, nullptr,
                          extra_out, ws, ws_bytes, stream);
}

int exsum_bdbs_finish(const void* in, void* out, int dtype, int op, int d, const int64_t* ext,
                      const int64_t* box, const void* total, void* ws, size_t ws_bytes,
                      void* stream) {
  if (total && op == EXSUM_MAX) return fail(EXSUM_ECONFIG, "bdbsc requires an invertible monoid");
  return run_stage_device(1, dtype, op, d, ext, box, 0, 0, in, out, total, nullptr, ws, ws_bytes,
                          stream);
}

// ---- the box-complement tail of a 3-D array, per axis-0 shard (tail2d.cu) ----
// stage -1: eligibility only; 0: R2_own[i] = fold of R_own row i (n_own rows);
// 1: T_own = rows [x0, x0 + n_own) of BC(R, (k0, k1)) from R2 (all n0 rows) and
// R's rows [x0, x0 + n_own + halo) held at R (halo = min(k0 - 1, n0 - x0 - n_own)).
int exsum_shard_bc_tail(int stage, const void* R, const void* R2, void* out, int dtype, int op,
                        int64_t n0, int64_t n1, int64_t k0, int64_t k1, int64_t x0, int64_t n_own,
                        void* stream) {
  g_err.clear();
  int rc = check_types(dtype, op);
  if (rc) return rc;
  if (n0 < 1 || n1 < 1 || k0 < 1 || k1 < 1) return fail(EXSUM_EUSAGE, "bad extents or box");
  if (x0 < 0 || n_own < 0 || x0 + n_own > n0) return fail(EXSUM_EUSAGE, "rows out of range");
  if (!tail2d_ok(dtype, n0, n1, k0)) return fail(EXSUM_ECONFIG, "no shard tail kernel for this shape");
  if (stage < 0) return EXSUM_OK;
  if (n_own == 0) {
    g_last_launches = 0;
    return EXSUM_OK;
  }
  const int64_t kk0 = k0 < n0 ? k0 : n0, kk1 = k1 < n1 ? k1 : n1;
  const size_t es = dtype_size(dtype);
  int n = 0;
  if (stage == 0) {
    if (!R || !out) return fail(EXSUM_EUSAGE, "null buffer");
    n = launch_tail2d_shard(dtype, op, const_cast<void*>(R), out, nullptr, n0, n1, kk0, kk1, 0, n_own,
                            (cudaStream_t)stream, 0);
  } else {
    if (!R || !R2 || !out) return fail(EXSUM_EUSAGE, "null buffer");
    // R and out addressed by the global row: shift the bases back by x0 rows
    const char* rv = static_cast<const char*>(R) - (size_t)(x0 * n1) * es;
    char* ov = static_cast<char*>(out) - (size_t)(x0 * n1) * es;
    n = launch_tail2d_shard(dtype, op, rv, const_cast<void*>(R2), ov, n0, n1, kk0, kk1, x0,
                            x0 + n_own, (cudaStream_t)stream, 1);
  }
  if (n < 0) return fail(EXSUM_ECONFIG, "no shard tail kernel for this dtype/operator");
  g_last_launches = n;
  g_total_launches += n;
  return cuda_check("shard tail");
}

// ---- box-complement for max as marginals, sharded along axis 0 (idem_max.cu) ----
static int idem_shard_check(int dtype, int op, int d, const int64_t* ext, int64_t x0,
                            int64_t n_own) {
  int rc = check_types(dtype, op);
  if (rc) return rc;
  if (d < 1 || d > EXSUM_MAX_DIMS || !ext) return fail(EXSUM_EUSAGE, "bad extents");
  for (int i = 0; i < d; ++i)
    if (ext[i] < 1) return fail(EXSUM_EUSAGE, "every extent must be >= 1");
  if (x0 < 0 || n_own < 0 || x0 + n_own > ext[0]) return fail(EXSUM_EUSAGE, "planes out of range");
  if (!idem_max_ok(dtype, op, d, ext))
    return fail(EXSUM_ECONFIG, "the marginal form needs max over int64, d >= 2 and sum(ext) <= 4096");
  return EXSUM_OK;
}

int exsum_shard_idem_workspace_bytes(int dtype, int op, int d, const int64_t* ext, size_t* bytes) {
  g_err.clear();
  int rc = idem_shard_check(dtype, op, d, ext, 0, 0);
  if (rc) return rc;
  int64_t S = 0;
  for (int i = 0; i < d; ++i) S += ext[i];
  if (bytes) *bytes = (size_t)S * 8;
  return EXSUM_OK;
}

int exsum_shard_idem_marginals(const void* in, void* marg, int dtype, int op, int d,
                               const int64_t* ext, int64_t x0, int64_t n_own, void* ws,
                               size_t ws_bytes, void* stream) {
  g_err.clear();
  int rc = idem_shard_check(dtype, op, d, ext, x0, n_own);
  if (rc) return rc;
  if (!marg || (n_own > 0 && !in)) return fail(EXSUM_EUSAGE, "null buffer");
  size_t need = 0;
  int64_t k1[EXSUM_MAX_DIMS];
  for (int i = 0; i < d; ++i) k1[i] = 1;
  launch_idem_max_shard(dtype, in, nullptr, marg, d, ext, k1, x0, n_own, nullptr, &need, nullptr, -1);
  if (!ws || ws_bytes < need) return fail(EXSUM_EUSAGE, "workspace too small (see exsum_shard_idem_workspace_bytes)");
  const int n = launch_idem_max_shard(dtype, in, nullptr, marg, d, ext, k1, x0, n_own, ws, nullptr,
                                      (cudaStream_t)stream, 0);
  if (n < 0) return fail(EXSUM_ECUDA, "marginal kernels failed to launch");
  g_last_launches = n;
  g_total_launches += n;
  return cuda_check("shard marginals");
}

int exsum_shard_idem_write(const void* marg, void* out, int dtype, int op, int d, const int64_t* ext,
                           const int64_t* box, int64_t x0, int64_t n_own, void* stream) {
  g_err.clear();
  int rc = idem_shard_check(dtype, op, d, ext, x0, n_own);
  if (rc) return rc;
  Shape sh;
  rc = normalize(d, ext, box, &sh);
  if (rc) return rc;
  if (!marg || (n_own > 0 && !out)) return fail(EXSUM_EUSAGE, "null buffer");
  if (n_own == 0) {
    g_last_launches = 0;
    return EXSUM_OK;
  }
  const int n = launch_idem_max_shard(dtype, nullptr, out, const_cast<void*>(marg), d, ext, sh.k, x0,
                                      n_own, nullptr, nullptr, (cudaStream_t)stream, 1);
  if (n < 0) return fail(EXSUM_ECUDA, "broadcast kernel failed to launch");
  g_last_launches = n;
  g_total_launches += n;
  return cuda_check("shard broadcast");
}

int exsum_box_complement_finish(const void* in, void* out, int dtype, int op, int d,
                                const int64_t* ext, const int64_t* box, const void* tail,
                                void* ws, size_t ws_bytes, void* stream) {
  if (!tail) return fail(EXSUM_EUSAGE, "tail is required");
  return run_stage_device(2, dtype, op, d, ext, box, 0, 0, in, out, tail, nullptr, ws, ws_bytes,
                          stream);
}

int exsum_release_cache(void) {
  release_graphs();
  {
    BatchCache& b = batch_cache();
    std::lock_guard<std::mutex> lock(b.mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (size_t i = 0; i < b.slots.size(); ++i) {
      cudaSetDevice(b.dev[i / 2]);
      b.slots[i].in.release();
      b.slots[i].out.release();
      b.slots[i].ws.release();
    }
    cudaSetDevice(cur);
  }
  HostCache& c = host_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (size_t i = 0; i < c.dev.size(); ++i) {
    cudaSetDevice(c.dev[i]);
    c.in[i].release();
    c.out[i].release();
    c.ws[i].release();
    cudaStreamDestroy(c.stream[i]);
  }
  cudaSetDevice(cur);
  c.dev.clear();
  c.in.clear();
  c.out.clear();
  c.ws.clear();
  c.stream.clear();
  return EXSUM_OK;
}

}  // extern "C"
