/*
 * exsum_b200.h -- C ABI of the B200-native box-sum library (libexsum_b200.so).
 *
 * Drop-in boundary for the reference's hot path (arxiv 2106.00124 `exsum`
 * package, /root/reference/pkg/src/exsum).  The reference is Python; its
 * plug-in surface is the set of callables `fn(t: Tensor, box) -> Tensor`
 * registered in bench.ALGORITHMS (bench.py:60-76) plus bdbs_1d (scan.py:53).
 * Each entry point below replaces one of them; the Python host layer
 * (paper_2106_00124_b200/) binds them with ctypes exactly as a maintainer of
 * the reference would.
 *
 * Conventions:
 *   - arrays are dense C-order (last axis contiguous), same
 *     extents and dtype in and out; `in` is never written; out != in;
 *   - box sides are clamped to the extents (tensor.py:32-48); windows are
 *     forward, half-open, clipped at the end;
 *   - work is stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream); the call returns after enqueueing;
 *   - no hidden device allocations on the device-pointer entry points: the
 *     caller passes a workspace of exsum_workspace_bytes() bytes (enough for
 *     16-byte aligned arrays, as every CUDA allocation is, and for arrays off
 *     that alignment, which run unfused kernels);
 *   - no CPU fallback: an unsupported dtype/operator is EXSUM_ECONFIG.
 *
 * Return codes map onto the reference's exceptions (errors.py:8-22):
 *   EXSUM_OK 0, EXSUM_EUSAGE 1 (UsageError: bad extents / box arity / k < 1),
 *   EXSUM_ECONFIG 2 (ConfigurationError: e.g. weak route on max),
 *   EXSUM_ECUDA 3 (CUDA runtime failure; see exsum_last_error()).
 */
#ifndef EXSUM_B200_H
#define EXSUM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EXSUM_ABI_VERSION 2

/* element types (MonoidOps.dtype, monoid.py:40) */
#define EXSUM_F32 0 /* add-f32 (test-side float32 FloatAddOps)      */
#define EXSUM_F64 1 /* add-f64  FloatAddOps   monoid.py:167-204      */
#define EXSUM_I64 2 /* add-i64 / max-i64 / mod-add:<m>  monoid.py:130-164,207-286 */

/* operators (MonoidOps.combine) */
#define EXSUM_ADD 0
#define EXSUM_MAX 1
#define EXSUM_MODADD 2 /* mod-add:<m> ModAddOps monoid.py:235-286; int64, needs the
                          modulus (2 <= m <= 2^31): only the exsum_route* calls take it */

/* routes (bench.ALGORITHMS names, bench.py:60-76) */
#define EXSUM_ROUTE_BDBS 0           /* "bdbs"           included.py:124-129 */
#define EXSUM_ROUTE_BDBSC 1          /* "bdbsc"          excluded.py:88-90   */
#define EXSUM_ROUTE_BOX_COMPLEMENT 2 /* "box-complement" excluded.py:129-159 */
#define EXSUM_ROUTE_SAT 3            /* "sat"            included.py:98-121  */
#define EXSUM_ROUTE_SATC 4           /* "satc"           excluded.py:83-85   */
#define EXSUM_ROUTE_CORNERS 5        /* "corners"        excluded.py:200-225 (2-D, 3-D) */
#define EXSUM_ROUTE_CORNERS_SPINE 6  /* "corners-spine"  excluded.py:228-262 (2-D, 3-D);
                                        same values as "corners" bit for bit */

#define EXSUM_OK 0
#define EXSUM_EUSAGE 1
#define EXSUM_ECONFIG 2
#define EXSUM_ECUDA 3

#define EXSUM_MAX_DIMS 32

/* ABI version of the loaded library (== EXSUM_ABI_VERSION). */
int exsum_abi_version(void);

/* Message for the last non-zero return on this thread ("" if none). */
const char *exsum_last_error(void);

/* Workspace bytes the route needs for these extents/box (validated like the
 * route itself).  Replaces the reference's hidden allocations
 * (alloc.new_array, alloc.py:63-65; tensor.py:91-114; scan.py:70). */
int exsum_workspace_bytes(int route, int dtype, int op, int d, const int64_t *ext,
                          const int64_t *box, size_t *bytes);

/* Any route (EXSUM_ROUTE_*) with any operator, including mod-add:<m>
 * (`modulus` is ignored for the other operators).  Replaces the registry slot
 * `fn(t, box)` of every bench.ALGORITHMS entry on this path (bench.py:60-76):
 * "bdbs", "bdbsc", "box-complement", "sat" (included.py:98-121), "satc"
 * (excluded.py:83-85), "corners" and "corners-spine" (excluded.py:191-262).
 * bdbsc / sat / satc need an invertible operator (add, mod-add); max returns
 * EXSUM_ECONFIG like bench.check_algorithm_config; corners need d in {2, 3}. */
int exsum_route(int route, const void *in, void *out, int dtype, int op, int64_t modulus, int d,
                const int64_t *ext, const int64_t *box, void *ws, size_t ws_bytes, void *stream);
int exsum_route_workspace_bytes(int route, int dtype, int op, int64_t modulus, int d,
                                const int64_t *ext, const int64_t *box, size_t *bytes);
/* Host-buffer form of exsum_route (see exsum_run_host). */
int exsum_route_host(int route, const void *h_in, void *h_out, int dtype, int op, int64_t modulus,
                     int d, const int64_t *ext, const int64_t *box);

/* Strong included sum, any monoid.  Replaces bdbs_included(t, box)
 * (included.py:124-129); bdbs_1d(ops, values, k) (scan.py:53-58) is d == 1. */
int exsum_bdbs_included(const void *in, void *out, int dtype, int op, int d,
                        const int64_t *ext, const int64_t *box, void *ws, size_t ws_bytes,
                        void *stream);

/* Weak excluded sum (total (-) included), invertible monoids only (add).
 * Replaces bdbs_excluded(t, box) (excluded.py:88-90, 72-75). */
int exsum_bdbsc_excluded(const void *in, void *out, int dtype, int op, int d,
                         const int64_t *ext, const int64_t *box, void *ws, size_t ws_bytes,
                         void *stream);

/* Strong excluded sum, any monoid.  Replaces box_complement_excluded(t, box)
 * (excluded.py:129-159). */
int exsum_box_complement_excluded(const void *in, void *out, int dtype, int op, int d,
                                  const int64_t *ext, const int64_t *box, void *ws,
                                  size_t ws_bytes, void *stream);

/* One windowed pass along `axis` (out-of-place).  Replaces
 * windowed_sum_axis(ops, view, k, axis) (scan.py:61-102) on a dense array. */
int exsum_windowed_pass(const void *in, void *out, int dtype, int op, int d,
                        const int64_t *ext, int axis, int64_t k, void *stream);

/* ---- building blocks, device arrays, stream-ordered ----
 * op: EXSUM_ADD / EXSUM_MAX / EXSUM_MODADD (with `modulus`). */

/* MonoidOps.accumulate(arr, axis, reverse) (monoid.py:156-159, 196-198, 224-226,
 * 280-283) out of place or in place (in == out): a sequential running fold
 * along `axis` -- and with it prefix_along_dim / suffix_along_dim
 * (scan.py:113-120) on a reduced slice. */
int exsum_scan_workspace_bytes(int dtype, int op, int64_t modulus, int d, const int64_t *ext,
                               int axis, size_t *bytes);
int exsum_scan_axis(const void *in, void *out, int dtype, int op, int64_t modulus, int d,
                    const int64_t *ext, int axis, int reverse, void *ws, size_t ws_bytes,
                    void *stream);

/* add_contribution(src, dst, dim, offset) (excluded.py:111-126): dst has extents
 * ext; src is the reduced slice of shape ext[dim:]; dst[.., x_dim, ..] (+)=
 * src[x_dim + offset, ..] wherever 0 <= x_dim + offset < ext[dim]. */
int exsum_add_contribution(const void *src, void *dst, int dtype, int op, int64_t modulus, int d,
                           const int64_t *ext, int dim, int64_t offset, void *stream);

/* MonoidOps bulk kernels on n elements: kind 0 combine_into(dst, src) (also
 * rcombine_into: every operator is commutative), 1 subtract_into(dst, src),
 * 2 rsubtract_scalar(*scalar, dst) with `scalar` a host pointer to one element.
 * Kinds 1 and 2 need an inverse (EXSUM_ECONFIG for max). */
int exsum_elementwise(void *dst, const void *src, const void *scalar, int dtype, int op,
                      int64_t modulus, int kind, int64_t n, void *stream);

/* MonoidOps.fold (monoid.py:161-164, 200-204, 229-232, 284-286) of n elements into
 * one element of device memory `result` (deterministic tree; float32 accumulates
 * in float64; the identity when n == 0). */
size_t exsum_fold_workspace_bytes(void);
int exsum_fold(const void *in, void *result, int dtype, int op, int64_t modulus, int64_t n,
               void *ws, size_t ws_bytes, void *stream);

/* Host-buffer convenience: copies h_in to the device, runs `route`, copies
 * the result to h_out and synchronizes.  Device buffers are cached per
 * device between calls.  This is the call a host-side plug-in makes
 * (AlgorithmInfo.run with numpy data, bench.py:54-57). */
int exsum_run_host(int route, const void *h_in, void *h_out, int dtype, int op, int d,
                   const int64_t *ext, const int64_t *box);

/* A stream of `count` independent arrays of the same extents through one route
 * (AlgorithmInfo.run over many inputs): h_in[i] -> h_out[i].  Two device slots
 * and separate copy streams pipeline the host->device copy of array i+1, the
 * compute of array i and the device->host copy of array i-1 (the copy engines
 * run both directions at once).  Returns after the last copy lands.  Pinned
 * host buffers give full PCIe bandwidth. */
int exsum_route_host_batch(int route, int count, const void *const *h_in, void *const *h_out,
                           int dtype, int op, int64_t modulus, int d, const int64_t *ext,
                           const int64_t *box);

/* Release the device buffers cached by exsum_run_host / exsum_route_host_batch. */
int exsum_release_cache(void);

/* Number of kernels the last successful call on this thread launched
 * (instrumentation for bench.py's gpu_launches). */
int exsum_last_launch_count(void);

/* Cumulative number of kernels launched by this library on this thread. */
long long exsum_total_launch_count(void);

/* Per-kernel CUDA-event profiling of the calls made on this thread (for
 * bench.py's roofline): enable (clears old records), run, synchronize, then
 * read each launch's name, algorithmic bytes (compulsory reads + writes) and
 * device time in milliseconds. */
int exsum_profile_enable(int on);
int exsum_profile_count(void);
int exsum_profile_get(int i, char *name, int name_len, double *bytes, float *ms);

/* ---- axis-0 sharding stages (multi-GPU; no NCCL inside) ----
 * A rank owns planes [x_s, x_e) of axis 0 (x_s a multiple of box[0]) and holds
 * the next rank's first box[0]-1 planes as a halo right after them.
 *
 * exsum_shard_axis0_pass: the axis-0 windowed pass of own+halo planes
 *   (ext_in[0] = own + halo) producing only the n_out own planes; extra_kind
 *   1 also writes R (fold over the last axis of the own raw planes,
 *   n_out*prod(ext[1:d-1]) elements), 2 the local total (one double for
 *   float types, one int64 for add-i64) into extra_out.
 * exsum_bdbs_finish: the remaining windowed passes (axes 1..d-1) of a shard;
 *   total != NULL (device, the global total) applies the BDBSC complement.
 * exsum_box_complement_finish: the remaining W passes (axes 1..d-2) and the
 *   last-axis round with the tail slice (device, one value per own row). */
int exsum_shard_workspace_bytes(int stage, int dtype, int op, int d, const int64_t *ext,
                                const int64_t *box, int64_t n_out, int extra_kind,
                                size_t *bytes);
int exsum_shard_axis0_pass(const void *in, void *out, int dtype, int op, int d,
                           const int64_t *ext_in, const int64_t *box, int64_t n_out,
                           int extra_kind, void *extra_out, void *ws, size_t ws_bytes,
                           void *stream);
int exsum_bdbs_finish(const void *in, void *out, int dtype, int op, int d, const int64_t *ext,
                      const int64_t *box, const void *total, void *ws, size_t ws_bytes,
                      void *stream);
int exsum_box_complement_finish(const void *in, void *out, int dtype, int op, int d,
                                const int64_t *ext, const int64_t *box, const void *tail,
                                void *ws, size_t ws_bytes, void *stream);

/* The box-complement tail of a 3-D array per axis-0 shard (R = fold over the
 * last axis, n0 x n1; T = BC(R, (k0, k1)); a rank holds rows [x0, x0 + n_own)):
 * stage 0 folds the rank's R rows into R2_own (out, n_own values); stage 1
 * writes the rank's T rows (out, n_own x n1) from the all-gathered R2 (n0
 * values) and R's rows [x0, x0 + n_own + min(k0 - 1, n0 - x0 - n_own)) (the
 * rank's own and the next rank's first k0 - 1, at R); stage -1 checks
 * eligibility only (EXSUM_ECONFIG: use the all-gathered R and the full route). */
int exsum_shard_bc_tail(int stage, const void *R, const void *R2, void *out, int dtype, int op,
                        int64_t n0, int64_t n1, int64_t k0, int64_t k1, int64_t x0, int64_t n_own,
                        void *stream);

/* Box-complement for max (int64) as per-axis marginals, sharded along axis 0
 * (no halo: the ranks all-reduce sum(ext) values).  ext is the GLOBAL extents;
 * a rank holds global planes [x0, x0 + n_own).
 * exsum_shard_idem_marginals: the rank's marginals M_a[i] (max over the
 *   rank's elements with coordinate i on axis a; INT64_MIN where it has none)
 *   into marg (sum(ext) int64, device); workspace sum(ext) * 8 bytes.
 * exsum_shard_idem_write: the rank's output planes from the all-reduced
 *   (elementwise max over ranks) marginals.
 * EXSUM_ECONFIG when the form does not apply (not max-i64, d < 2 or
 * sum(ext) > 4096): run the slab stages above instead. */
int exsum_shard_idem_workspace_bytes(int dtype, int op, int d, const int64_t *ext, size_t *bytes);
int exsum_shard_idem_marginals(const void *in, void *marg, int dtype, int op, int d,
                               const int64_t *ext, int64_t x0, int64_t n_own, void *ws,
                               size_t ws_bytes, void *stream);
int exsum_shard_idem_write(const void *marg, void *out, int dtype, int op, int d,
                           const int64_t *ext, const int64_t *box, int64_t x0, int64_t n_own,
                           void *stream);

#ifdef __cplusplus
}
#endif

#endif /* EXSUM_B200_H */
