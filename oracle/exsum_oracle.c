/*
 * exsum_oracle.c -- CPU restatement of the reference box-sum path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2106_00124_b200/csrc).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it.
 *
 * It restates, with the reference's exact floating-point association, the
 * algorithms in /root/reference/pkg/src/exsum:
 *   - windowed_sum_axis          scan.py:61-102   (oracle_win_line)
 *   - bdbs_included              included.py:124-129
 *   - bdbs_excluded (+ fold,     excluded.py:72-75, 88-90; monoid.py:161-164,
 *     rsubtract_scalar)          200-204, 154-155, 193-194
 *   - box_complement_excluded    excluded.py:129-159 (+ add_contribution :111-126,
 *                                reduced_slice/prefix/suffix scan.py:105-120)
 *   - oracle_included/excluded   oracle.py:37-71 (brute force, row-major fold)
 * Pinning: tests/test_oracle.py checks every function here against golden
 * vectors produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Lines are independent, so the per-line loops run under OpenMP; the result
 * does not depend on the thread count (each line is computed sequentially in
 * the reference's order).  The BDBSC total is a single sequential fold, as
 * in the reference.
 *
 *   - sat_included / sat_excluded included.py:37-121, excluded.py:83-85
 *   - mod-add:<m> monoid           monoid.py:235-286 (op code 2, oracle_set_modulus)
 *   - corners / corners-spine      excluded.py:41-66, 191-292 (2-D, 3-D)
 *
 * dtype codes: 0 = float32, 1 = float64, 2 = int64.  op codes: 0 = add, 1 = max,
 * 2 = mod-add.
 * Return codes: 0 ok, 1 usage error, 2 configuration error.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_USAGE 1
#define ORC_CONFIG 2
/* column tile of the strided passes (elements) */
#define ORC_TILE 256

/* memcpy split over the OpenMP threads (large buffers: first touch and copy in parallel) */
static void pcopy(void *dst, const void *src, size_t bytes) {
    const size_t CH = (size_t)1 << 20;
    int64_t nch = (int64_t)((bytes + CH - 1) / CH);
    _Pragma("omp parallel for schedule(static)")
    for (int64_t c = 0; c < nch; ++c) {
        size_t o = (size_t)c * CH, b = bytes - o < CH ? bytes - o : CH;
        memcpy((char *)dst + o, (const char *)src + o, b);
    }
}

static int64_t prod_range(const int64_t *ext, int lo, int hi) {
    int64_t p = 1;
    for (int i = lo; i < hi; ++i) p *= ext[i];
    return p;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

/* int64 addition wraps mod 2^64 like numpy (monoid.py:161-164). */
static inline int64_t i64_add(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
static inline int64_t i64_sub(int64_t a, int64_t b) { return (int64_t)((uint64_t)a - (uint64_t)b); }

/*
 * One instantiation per (type, operator).  C(a,b) is the monoid combine
 * (combine_into / rcombine_into); the reference applies it as np.add(dst, src)
 * / np.maximum(dst, src), and both are commutative, so operand order inside
 * one combine never changes the bits.  ACC(a,b) and FIN(v) restate
 * MonoidOps.accumulate: a running ACC along the line, then FIN on every
 * element of it (identity for the plain monoids; for mod-add a raw int64
 * cumsum followed by np.remainder over the whole line, monoid.py:280-283,
 * so even an element no combine touched comes out reduced).
 */
#define DEFINE_ORACLE(SFX, T, C, ACC, FIN, IDENT)                                              \
    /* scan.py:61-102 -- in-place windowed sum of one strided line. */                         \
    static void win_line_##SFX(T *buf, int64_t n, int64_t stride, int64_t k, T *scratch) {    \
        if (n == 0 || k == 1) return;                                                          \
        if (k >= n) { /* scan.py:66-68: reverse inclusive scan (ops.accumulate) */            \
            for (int64_t x = n - 2; x >= 0; --x)                                               \
                buf[x * stride] = ACC(buf[x * stride], buf[(x + 1) * stride]);                 \
            for (int64_t x = 0; x < n; ++x) buf[x * stride] = FIN(buf[x * stride]);            \
            return;                                                                            \
        }                                                                                      \
        for (int64_t x = 0; x < n; ++x) scratch[x] = buf[x * stride];                          \
        for (int64_t bs = 0; bs < n; bs += k) {                                                \
            int64_t be = bs + k < n ? bs + k : n;                                              \
            /* in-block suffix, right nested (scan.py:75-79) */                               \
            for (int64_t x = be - 2; x >= bs; --x)                                             \
                buf[x * stride] = C(buf[x * stride], buf[(x + 1) * stride]);                   \
            /* in-block prefix on the scratch copy, left nested (scan.py:82-86) */            \
            for (int64_t x = bs + 1; x < be; ++x) scratch[x] = C(scratch[x], scratch[x - 1]);  \
        }                                                                                      \
        /* stitch (scan.py:88-102): off block starts, outside the last block */              \
        int64_t last_bs = k * ((n - 1) / k);                                                   \
        for (int64_t x = 1; x < last_bs; ++x) {                                                \
            if (x % k == 0) continue;                                                          \
            int64_t p = x + k - 1 < n - 1 ? x + k - 1 : n - 1;                                 \
            buf[x * stride] = C(buf[x * stride], scratch[p]);                                  \
        }                                                                                      \
    }                                                                                          \
                                                                                               \
    /* win_line_ on W adjacent lines at once (columns c of a strided axis): the same */      \
    /* operations in the same order per column, walked row by row so every access */          \
    /* is a contiguous run of W elements (cache lines used whole, vectorisable). */            \
    static void win_tile_##SFX(T *buf, int64_t n, int64_t stride, int64_t k, int64_t W,       \
                               T *scratch) {                                                   \
        if (n == 0 || k == 1) return;                                                          \
        if (k >= n) {                                                                          \
            for (int64_t x = n - 2; x >= 0; --x) {                                             \
                T *r = buf + x * stride; const T *q = r + stride;                              \
                for (int64_t c = 0; c < W; ++c) r[c] = ACC(r[c], q[c]);                        \
            }                                                                                  \
            for (int64_t x = 0; x < n; ++x) {                                                  \
                T *r = buf + x * stride;                                                       \
                for (int64_t c = 0; c < W; ++c) r[c] = FIN(r[c]);                              \
            }                                                                                  \
            return;                                                                            \
        }                                                                                      \
        for (int64_t x = 0; x < n; ++x) memcpy(scratch + x * W, buf + x * stride, sizeof(T) * (size_t)W); \
        for (int64_t bs = 0; bs < n; bs += k) {                                                \
            int64_t be = bs + k < n ? bs + k : n;                                              \
            for (int64_t x = be - 2; x >= bs; --x) {                                           \
                T *r = buf + x * stride; const T *q = r + stride;                              \
                for (int64_t c = 0; c < W; ++c) r[c] = C(r[c], q[c]);                          \
            }                                                                                  \
            for (int64_t x = bs + 1; x < be; ++x) {                                            \
                T *r = scratch + x * W; const T *q = r - W;                                    \
                for (int64_t c = 0; c < W; ++c) r[c] = C(r[c], q[c]);                          \
            }                                                                                  \
        }                                                                                      \
        int64_t last_bs = k * ((n - 1) / k);                                                   \
        for (int64_t x = 1; x < last_bs; ++x) {                                                \
            if (x % k == 0) continue;                                                          \
            int64_t p = x + k - 1 < n - 1 ? x + k - 1 : n - 1;                                 \
            T *r = buf + x * stride; const T *q = scratch + p * W;                             \
            for (int64_t c = 0; c < W; ++c) r[c] = C(r[c], q[c]);                              \
        }                                                                                      \
    }                                                                                          \
                                                                                               \
    /* windowed_sum_axis over every line of a C-order array [outer, n, inner]. */             \
    /* Contiguous lines (inner == 1) one per iteration; strided lines in tiles of */          \
    /* ORC_TILE adjacent columns (bit-identical: every column keeps its own order). */        \
    static void pass_##SFX(T *data, int64_t outer, int64_t n, int64_t inner, int64_t k) {     \
        if (k == 1 || n == 0) return;                                                          \
        if (inner == 1) {                                                                      \
            _Pragma("omp parallel")                                                            \
            {                                                                                  \
                T *scratch = (T *)malloc(sizeof(T) * (size_t)n);                               \
                _Pragma("omp for schedule(static)")                                            \
                for (int64_t o = 0; o < outer; ++o) win_line_##SFX(data + o * n, n, 1, k, scratch); \
                free(scratch);                                                                 \
            }                                                                                  \
            return;                                                                            \
        }                                                                                      \
        int64_t tiles = (inner + ORC_TILE - 1) / ORC_TILE;                                     \
        _Pragma("omp parallel")                                                                \
        {                                                                                      \
            T *scratch = (T *)malloc(sizeof(T) * (size_t)n * ORC_TILE);                        \
            _Pragma("omp for schedule(static)")                                                \
            for (int64_t l = 0; l < outer * tiles; ++l) {                                      \
                int64_t o = l / tiles, c0 = (l % tiles) * ORC_TILE;                            \
                int64_t W = inner - c0 < ORC_TILE ? inner - c0 : ORC_TILE;                     \
                win_tile_##SFX(data + o * n * inner + c0, n, inner, k, W, scratch);            \
            }                                                                                  \
            free(scratch);                                                                     \
        }                                                                                      \
    }                                                                                          \
                                                                                               \
    /* np.add.accumulate / np.maximum.accumulate along axis 0 of [n, m] (forward or */        \
    /* flipped); sequential per column like numpy, walked in column tiles. */                 \
    static void axis0_scan_##SFX(T *s, int64_t n, int64_t m, int reverse) {                    \
        int64_t tiles = (m + ORC_TILE - 1) / ORC_TILE;                                         \
        _Pragma("omp parallel for schedule(static)")                                           \
        for (int64_t t = 0; t < tiles; ++t) {                                                  \
            int64_t c0 = t * ORC_TILE, c1 = c0 + ORC_TILE < m ? c0 + ORC_TILE : m;             \
            if (!reverse) {                                                                    \
                for (int64_t x = 1; x < n; ++x)                                                \
                    for (int64_t c = c0; c < c1; ++c) s[x * m + c] = ACC(s[(x - 1) * m + c], s[x * m + c]); \
            } else {                                                                           \
                for (int64_t x = n - 2; x >= 0; --x)                                           \
                    for (int64_t c = c0; c < c1; ++c) s[x * m + c] = ACC(s[(x + 1) * m + c], s[x * m + c]); \
            }                                                                                  \
            for (int64_t x = 0; x < n; ++x)                                                    \
                for (int64_t c = c0; c < c1; ++c) s[x * m + c] = FIN(s[x * m + c]);            \
        }                                                                                      \
    }                                                                                          \
                                                                                               \
    static void bdbs_##SFX(const T *in, T *out, int d, const int64_t *ext, const int64_t *k) { \
        int64_t N = prod_range(ext, 0, d);                                                     \
        pcopy(out, in, sizeof(T) * (size_t)N);                                                 \
        for (int a = 0; a < d; ++a)                                                            \
            pass_##SFX(out, prod_range(ext, 0, a), ext[a], prod_range(ext, a + 1, d), k[a]);   \
    }                                                                                          \
                                                                                               \
    /* MonoidOps.fold: strict row-major left fold (monoid.py:161-164,200-204,229-232). */     \
    static inline T fold_##SFX(const T *a, int64_t N) {                                        \
        if (N == 0) return (T)(IDENT);                                                         \
        T acc = a[0];                                                                          \
        for (int64_t i = 1; i < N; ++i) acc = C(acc, a[i]);                                    \
        return acc;                                                                            \
    }                                                                                          \
                                                                                               \
    /* excluded.py:111-126: out[.., x_dim, ..] (+)= src[x_dim + offset, ..] in range, */      \
    /* broadcast over the dims before dim.  src is the reduced slice (shape ext[dim:]). */     \
    static void add_contribution_##SFX(const T *src, T *out, int d, const int64_t *ext,       \
                                       int dim, int64_t offset) {                              \
        int64_t outer = prod_range(ext, 0, dim), n = ext[dim], inner = prod_range(ext, dim + 1, d); \
        int64_t lo = offset < 0 ? -offset : 0;                                                 \
        int64_t hi = n - offset < n ? n - offset : n;                                          \
        if (lo >= hi) return;                                                                  \
        _Pragma("omp parallel for collapse(2) schedule(static)")                               \
        for (int64_t o = 0; o < outer; ++o)                                                    \
            for (int64_t x = lo; x < hi; ++x) {                                                \
                T *dst = out + (o * n + x) * inner;                                            \
                const T *s = src + (x + offset) * inner;                                       \
                for (int64_t m = 0; m < inner; ++m) dst[m] = C(dst[m], s[m]);                  \
            }                                                                                  \
    }                                                                                          \
                                                                                               \
    /* excluded.py:129-159, literally (same buffers, same accumulation order). */            \
    static int box_complement_##SFX(const T *in, T *out, int d, const int64_t *ext,            \
                                    const int64_t *k) {                                        \
        int64_t N = prod_range(ext, 0, d);                                                     \
        T *cur = (T *)malloc(sizeof(T) * (size_t)N), *nxt = (T *)malloc(sizeof(T) * (size_t)N); \
        T *win = (T *)malloc(sizeof(T) * (size_t)N), *pre = (T *)malloc(sizeof(T) * (size_t)N); \
        if (!cur || !nxt || !win || !pre) {                                                    \
            free(cur); free(nxt); free(win); free(pre);                                        \
            return ORC_USAGE;                                                                  \
        }                                                                                      \
        _Pragma("omp parallel for schedule(static)")                                           \
        for (int64_t i = 0; i < N; ++i) { out[i] = (T)(IDENT); cur[i] = in[i]; }               \
        for (int i = 0; i < d; ++i) {                                                          \
            /* reduced_slice: dims < i pinned at their last index (scan.py:105-110) */        \
            int64_t off = 0, stride = N;                                                       \
            for (int j = 0; j < i; ++j) { stride /= ext[j]; off += (ext[j] - 1) * stride; }    \
            int64_t M = prod_range(ext, i, d), ni = ext[i], m = M / ni;                        \
            if (i < d - 1) {                                                                   \
                pcopy(nxt + off, cur + off, sizeof(T) * (size_t)M);                           \
                axis0_scan_##SFX(nxt + off, ni, m, 0);                                         \
            }                                                                                  \
            pcopy(win + off, cur + off, sizeof(T) * (size_t)M);                               \
            for (int j = i + 1; j < d; ++j)                                                    \
                pass_##SFX(win + off, prod_range(ext, i, j), ext[j], prod_range(ext, j + 1, d), k[j]); \
            pcopy(pre + off, win + off, sizeof(T) * (size_t)M);                               \
            axis0_scan_##SFX(pre + off, ni, m, 0);                                             \
            add_contribution_##SFX(pre + off, out, d, ext, i, -1);                             \
            axis0_scan_##SFX(win + off, ni, m, 1);                                             \
            add_contribution_##SFX(win + off, out, d, ext, i, k[i]);                           \
            if (i < d - 1) { T *t = cur; cur = nxt; nxt = t; }                                 \
        }                                                                                      \
        free(cur); free(nxt); free(win); free(pre);                                            \
        return ORC_OK;                                                                         \
    }                                                                                          \
                                                                                               \
    /* oracle.py:37-52 -- brute-force included sum, fold in row-major window order. */        \
    static void brute_inc_##SFX(const T *a, T *out, int d, const int64_t *ext, const int64_t *k) { \
        int64_t N = prod_range(ext, 0, d);                                                     \
        _Pragma("omp parallel for schedule(dynamic, 16)")                                      \
        for (int64_t f = 0; f < N; ++f) {                                                      \
            int64_t x[16], y[16], hi[16], str[16];                                             \
            int64_t r = f;                                                                     \
            for (int j = d - 1; j >= 0; --j) { x[j] = r % ext[j]; r /= ext[j]; }               \
            str[d - 1] = 1;                                                                    \
            for (int j = d - 2; j >= 0; --j) str[j] = str[j + 1] * ext[j + 1];                 \
            for (int j = 0; j < d; ++j) { y[j] = x[j]; hi[j] = x[j] + k[j] < ext[j] ? x[j] + k[j] : ext[j]; } \
            int have = 0;                                                                      \
            T acc = (T)(IDENT);                                                                \
            for (;;) {                                                                         \
                int64_t idx = 0;                                                               \
                for (int j = 0; j < d; ++j) idx += y[j] * str[j];                              \
                if (!have) { acc = a[idx]; have = 1; } else acc = C(acc, a[idx]);              \
                int j = d - 1;                                                                 \
                while (j >= 0) { if (++y[j] < hi[j]) break; y[j] = x[j]; --j; }               \
                if (j < 0) break;                                                              \
            }                                                                                  \
            out[f] = acc;                                                                      \
        }                                                                                      \
    }                                                                                          \
                                                                                               \
    /* oracle.py:55-71 -- brute-force excluded sum over the complement, row-major. */         \
    static void brute_exc_##SFX(const T *a, T *out, int d, const int64_t *ext, const int64_t *k) { \
        int64_t N = prod_range(ext, 0, d);                                                     \
        _Pragma("omp parallel for schedule(dynamic, 16)")                                      \
        for (int64_t f = 0; f < N; ++f) {                                                      \
            int64_t x[16], y[16];                                                              \
            int64_t r = f;                                                                     \
            for (int j = d - 1; j >= 0; --j) { x[j] = r % ext[j]; r /= ext[j]; }               \
            for (int j = 0; j < d; ++j) y[j] = 0;                                              \
            int have = 0;                                                                      \
            T acc = (T)(IDENT);                                                                \
            for (int64_t g = 0; g < N; ++g) {                                                  \
                int inside = 1;                                                                \
                for (int j = 0; j < d; ++j)                                                    \
                    if (!(x[j] <= y[j] && y[j] < x[j] + k[j])) { inside = 0; break; }          \
                if (!inside) { if (!have) { acc = a[g]; have = 1; } else acc = C(acc, a[g]); } \
                for (int j = d - 1; j >= 0; --j) { if (++y[j] < ext[j]) break; y[j] = 0; }     \
            }                                                                                  \
            out[f] = acc;                                                                      \
        }                                                                                      \
    }

/* mod-add:<m> (monoid.py:235-286): np.add / np.subtract on int64 (wrapping),
 * then np.remainder, which for m > 0 is the floor modulus in [0, m). */
static int64_t g_mod = 2;
static inline int64_t floor_mod(int64_t v) {
    int64_t r = v % g_mod;
    return r < 0 ? r + g_mod : r;
}
static inline int64_t mod_add(int64_t a, int64_t b) { return floor_mod(i64_add(a, b)); }
static inline int64_t mod_sub(int64_t a, int64_t b) { return floor_mod(i64_sub(a, b)); }

#define C_FADD(a, b) ((a) + (b))
#define C_FSUB(a, b) ((a) - (b))
#define C_IADD(a, b) i64_add((a), (b))
#define C_ISUB(a, b) i64_sub((a), (b))
#define C_MAX(a, b) ((a) >= (b) ? (a) : (b))
#define C_NOFIN(v) (v)

DEFINE_ORACLE(f32_add, float, C_FADD, C_FADD, C_NOFIN, 0.0f)
DEFINE_ORACLE(f64_add, double, C_FADD, C_FADD, C_NOFIN, 0.0)
DEFINE_ORACLE(i64_add, int64_t, C_IADD, C_IADD, C_NOFIN, 0)
DEFINE_ORACLE(i64_max, int64_t, C_MAX, C_MAX, C_NOFIN, INT64_MIN)
DEFINE_ORACLE(i64_mod, int64_t, mod_add, i64_add, floor_mod, 0)

/*
 * Summed-area-table routes, invertible monoids only (included.py:37-121,
 * excluded.py:83-85).  sat_build: copy, then ops.accumulate along axes
 * 0..d-1 in order (sequential per line, like numpy).  sat_included: out[x]
 * folds the 2^d corner terms of the identity-below / saturated-above query
 * table in itertools.product((False, True), repeat=d) order -- the all-high
 * corner is copied first, then each further term is combined (even number
 * of low picks) or subtracted (odd) into out, exactly like the numpy
 * combine_into / subtract_into sequence of sat_included.
 */
#define DEFINE_SAT(SFX, T, C, SUB, ACC, FIN, IDENT)                                            \
    static void sat_build_##SFX(const T *in, T *s, int d, const int64_t *ext) {               \
        int64_t N = prod_range(ext, 0, d);                                                     \
        memcpy(s, in, sizeof(T) * (size_t)N);                                                  \
        for (int a = 0; a < d; ++a) {                                                          \
            int64_t outer = prod_range(ext, 0, a), n = ext[a], inner = prod_range(ext, a + 1, d); \
            _Pragma("omp parallel for schedule(static)")                                       \
            for (int64_t l = 0; l < outer * inner; ++l) {                                      \
                T *line = s + (l / inner) * n * inner + (l % inner);                           \
                for (int64_t x = 1; x < n; ++x)                                                \
                    line[x * inner] = ACC(line[(x - 1) * inner], line[x * inner]);             \
                for (int64_t x = 0; x < n; ++x) line[x * inner] = FIN(line[x * inner]);        \
            }                                                                                  \
        }                                                                                      \
    }                                                                                          \
    static int sat_included_##SFX(const T *in, T *out, int d, const int64_t *ext,             \
                                  const int64_t *k) {                                          \
        int64_t N = prod_range(ext, 0, d);                                                     \
        T *s = (T *)malloc(sizeof(T) * (size_t)(N > 0 ? N : 1));                               \
        if (!s) return ORC_USAGE;                                                              \
        sat_build_##SFX(in, s, d, ext);                                                        \
        int64_t str[16];                                                                       \
        str[d - 1] = 1;                                                                        \
        for (int j = d - 2; j >= 0; --j) str[j] = str[j + 1] * ext[j + 1];                     \
        _Pragma("omp parallel for schedule(static)")                                           \
        for (int64_t f = 0; f < N; ++f) {                                                      \
            int64_t x[16];                                                                     \
            int64_t r = f;                                                                     \
            for (int j = d - 1; j >= 0; --j) { x[j] = r % ext[j]; r /= ext[j]; }               \
            T acc = (T)(IDENT);                                                                \
            for (int64_t p = 0; p < ((int64_t)1 << d); ++p) {                                  \
                int64_t idx = 0, lows = 0, below = 0;                                          \
                for (int j = 0; j < d; ++j) {                                                  \
                    int lo = (int)((p >> (d - 1 - j)) & 1);                                    \
                    int64_t c = lo ? x[j] - 1 : (x[j] + k[j] - 1 < ext[j] - 1 ? x[j] + k[j] - 1 : ext[j] - 1); \
                    lows += lo;                                                                \
                    if (c < 0) below = 1; else idx += c * str[j];                              \
                }                                                                              \
                T v = below ? (T)(IDENT) : s[idx];                                             \
                if (p == 0) acc = v;                                                           \
                else if (lows % 2 == 0) acc = C(acc, v);                                       \
                else acc = SUB(acc, v);                                                        \
            }                                                                                  \
            out[f] = acc;                                                                      \
        }                                                                                      \
        free(s);                                                                               \
        return ORC_OK;                                                                         \
    }

/*
 * Corner decompositions (excluded.py:41-66, 191-292): for every pattern in
 * sorted order ("PP" < "PS" < ...), a copy of A accumulated along axes
 * 0..d-1 in order -- forward for P, reversed for S (ops.accumulate) -- and
 * its contribution combined into the identity-filled output: along each
 * axis a prefix letter reads its scan at T-1 (clamped to n-1; nothing when
 * T-1 < 0) and a suffix letter at T (nothing when T >= n), with T = x (near
 * face) or x + k (far face) per the pattern's rule (CORNER_RULES,
 * excluded.py:45-62).  corners_excluded and corners_spine_excluded produce the
 * same scans and the same accumulation order, so one restatement serves both.
 */
static const char *const CORNER_KINDS2[4] = {"NF", "FF", "NN", "FN"};         /* PP PS SP SS */
static const char *const CORNER_KINDS3[8] = {"FNF", "FFF", "NNF", "NFF",
                                            "FNN", "FFN", "NNN", "NFN"};      /* PPP..SSS */

#define DEFINE_CORNERS(SFX, T, C, ACC, FIN, IDENT)                                             \
    static void line_scan_##SFX(T *s, int64_t outer, int64_t n, int64_t inner, int rev) {     \
        _Pragma("omp parallel for schedule(static)")                                           \
        for (int64_t l = 0; l < outer * inner; ++l) {                                          \
            T *line = s + (l / inner) * n * inner + (l % inner);                               \
            if (!rev) {                                                                        \
                for (int64_t x = 1; x < n; ++x)                                                \
                    line[x * inner] = ACC(line[(x - 1) * inner], line[x * inner]);             \
            } else {                                                                           \
                for (int64_t x = n - 2; x >= 0; --x)                                           \
                    line[x * inner] = ACC(line[(x + 1) * inner], line[x * inner]);             \
            }                                                                                  \
            for (int64_t x = 0; x < n; ++x) line[x * inner] = FIN(line[x * inner]);            \
        }                                                                                      \
    }                                                                                          \
    static int corners_##SFX(const T *in, T *out, int d, const int64_t *ext, const int64_t *k) { \
        if (d != 2 && d != 3) return ORC_CONFIG;                                               \
        int64_t N = prod_range(ext, 0, d);                                                     \
        T *sc = (T *)malloc(sizeof(T) * (size_t)N);                                            \
        if (!sc) return ORC_USAGE;                                                             \
        for (int64_t i = 0; i < N; ++i) out[i] = (T)(IDENT);                                   \
        int64_t str[3];                                                                        \
        str[d - 1] = 1;                                                                        \
        for (int j = d - 2; j >= 0; --j) str[j] = str[j + 1] * ext[j + 1];                     \
        for (int p = 0; p < (1 << d); ++p) {                                                   \
            const char *kinds = d == 2 ? CORNER_KINDS2[p] : CORNER_KINDS3[p];                  \
            memcpy(sc, in, sizeof(T) * (size_t)N);                                             \
            for (int a = 0; a < d; ++a) {                                                      \
                int suffix = (p >> (d - 1 - a)) & 1;                                           \
                line_scan_##SFX(sc, prod_range(ext, 0, a), ext[a], prod_range(ext, a + 1, d), suffix); \
            }                                                                                  \
            _Pragma("omp parallel for schedule(static)")                                       \
            for (int64_t f = 0; f < N; ++f) {                                                  \
                int64_t r = f, idx = 0;                                                        \
                int ok = 1;                                                                    \
                for (int a = d - 1; a >= 0; --a) {                                             \
                    int64_t x = r % ext[a];                                                    \
                    r /= ext[a];                                                               \
                    int suffix = (p >> (d - 1 - a)) & 1;                                       \
                    int64_t t = kinds[a] == 'N' ? x : x + k[a];                                \
                    int64_t src;                                                               \
                    if (!suffix) {                                                             \
                        if (t - 1 < 0) { ok = 0; break; }                                      \
                        src = t - 1 < ext[a] - 1 ? t - 1 : ext[a] - 1;                         \
                    } else {                                                                   \
                        if (t >= ext[a]) { ok = 0; break; }                                    \
                        src = t;                                                               \
                    }                                                                          \
                    idx += src * str[a];                                                       \
                }                                                                              \
                if (ok) out[f] = C(out[f], sc[idx]);                                           \
            }                                                                                  \
        }                                                                                      \
        free(sc);                                                                              \
        return ORC_OK;                                                                         \
    }

DEFINE_CORNERS(f32_add, float, C_FADD, C_FADD, C_NOFIN, 0.0f)
DEFINE_CORNERS(f64_add, double, C_FADD, C_FADD, C_NOFIN, 0.0)
DEFINE_CORNERS(i64_add, int64_t, C_IADD, C_IADD, C_NOFIN, 0)
DEFINE_CORNERS(i64_max, int64_t, C_MAX, C_MAX, C_NOFIN, INT64_MIN)
DEFINE_CORNERS(i64_mod, int64_t, mod_add, i64_add, floor_mod, 0)

DEFINE_SAT(f32_add, float, C_FADD, C_FSUB, C_FADD, C_NOFIN, 0.0f)
DEFINE_SAT(f64_add, double, C_FADD, C_FSUB, C_FADD, C_NOFIN, 0.0)
DEFINE_SAT(i64_add, int64_t, C_IADD, C_ISUB, C_IADD, C_NOFIN, 0)
DEFINE_SAT(i64_mod, int64_t, mod_add, mod_sub, i64_add, floor_mod, 0)

/* ---------------------------------------------------------------- C ABI --- */

/* tensor.py:20-48: extents >= 1, box arity, k >= 1, k clamped to n. */
static int normalize(int d, const int64_t *ext, const int64_t *box, int64_t *k) {
    if (d < 1 || d > 16) return ORC_USAGE;
    for (int i = 0; i < d; ++i) {
        if (ext[i] < 1 || box[i] < 1) return ORC_USAGE;
        k[i] = box[i] < ext[i] ? box[i] : ext[i];
    }
    return ORC_OK;
}

#define DISPATCH(FN, ...)                                                       \
    do {                                                                        \
        if (dtype == 0 && op == 0) { FN##_f32_add(__VA_ARGS__); break; }        \
        if (dtype == 1 && op == 0) { FN##_f64_add(__VA_ARGS__); break; }        \
        if (dtype == 2 && op == 0) { FN##_i64_add(__VA_ARGS__); break; }        \
        if (dtype == 2 && op == 1) { FN##_i64_max(__VA_ARGS__); break; }        \
        if (dtype == 2 && op == 2) { FN##_i64_mod(__VA_ARGS__); break; }        \
        return ORC_CONFIG;                                                      \
    } while (0)

int oracle_windowed_pass(void *data, int dtype, int op, int d, const int64_t *ext, int axis,
                         int64_t k, int nthreads) {
    if (d < 1 || axis < 0 || axis >= d || k < 1) return ORC_USAGE;
    set_threads(nthreads);
    int64_t outer = prod_range(ext, 0, axis), n = ext[axis], inner = prod_range(ext, axis + 1, d);
    if (k > n) k = n;
    DISPATCH(pass, data, outer, n, inner, k);
    return ORC_OK;
}

int oracle_bdbs_included(const void *in, void *out, int dtype, int op, int d,
                         const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    set_threads(nthreads);
    DISPATCH(bdbs, in, out, d, ext, k);
    return ORC_OK;
}

/* excluded.py:72-75,88-90: out = fold(A) (-) bdbs_included(A).  max has no
 * inverse -> configuration error (monoid.py:49-50). */
int oracle_bdbsc_excluded(const void *in, void *out, int dtype, int op, int d,
                          const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    if (op == 1) return ORC_CONFIG;
    set_threads(nthreads);
    int64_t N = prod_range(ext, 0, d);
    if (dtype == 0) {
        bdbs_f32_add(in, out, d, ext, k);
        /* FloatAddOps.fold: float(np.add.accumulate(arr)[-1]) is the float32
         * sequential fold; np.subtract(total, dst) keeps float32 (NEP 50). */
        float total = fold_f32_add(in, N);
        float *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = total - o[i];
    } else if (dtype == 1) {
        bdbs_f64_add(in, out, d, ext, k);
        double total = fold_f64_add(in, N);
        double *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = total - o[i];
    } else if (dtype == 2 && op == 0) {
        bdbs_i64_add(in, out, d, ext, k);
        int64_t total = fold_i64_add(in, N);
        int64_t *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = i64_sub(total, o[i]);
    } else if (dtype == 2 && op == 2) {
        /* ModAddOps.fold: int(arr.sum()) % m (wrapping int64 sum, floor mod);
         * rsubtract_scalar: np.subtract then np.remainder (monoid.py:274-286) */
        bdbs_i64_mod(in, out, d, ext, k);
        int64_t total = floor_mod(fold_i64_add(in, N));
        int64_t *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = mod_sub(total, o[i]);
    } else {
        return ORC_CONFIG;
    }
    return ORC_OK;
}

int oracle_box_complement_excluded(const void *in, void *out, int dtype, int op, int d,
                                   const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    set_threads(nthreads);
    if (dtype == 0 && op == 0) return box_complement_f32_add(in, out, d, ext, k);
    if (dtype == 1 && op == 0) return box_complement_f64_add(in, out, d, ext, k);
    if (dtype == 2 && op == 0) return box_complement_i64_add(in, out, d, ext, k);
    if (dtype == 2 && op == 1) return box_complement_i64_max(in, out, d, ext, k);
    if (dtype == 2 && op == 2) return box_complement_i64_mod(in, out, d, ext, k);
    return ORC_CONFIG;
}

/* "corners" / "corners-spine" (excluded.py:191-292), 2-D and 3-D only. */
int oracle_corners_excluded(const void *in, void *out, int dtype, int op, int d,
                            const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    set_threads(nthreads);
    if (dtype == 0 && op == 0) return corners_f32_add(in, out, d, ext, k);
    if (dtype == 1 && op == 0) return corners_f64_add(in, out, d, ext, k);
    if (dtype == 2 && op == 0) return corners_i64_add(in, out, d, ext, k);
    if (dtype == 2 && op == 1) return corners_i64_max(in, out, d, ext, k);
    if (dtype == 2 && op == 2) return corners_i64_mod(in, out, d, ext, k);
    return ORC_CONFIG;
}

/* mod-add:<m> modulus for op code 2 (2 <= m <= 2^31, monoid.py:27,250-256). */
int oracle_set_modulus(int64_t m) {
    if (m < 2 || m > ((int64_t)1 << 31)) return ORC_CONFIG;
    g_mod = m;
    return ORC_OK;
}

/* "sat" (included.py:98-121); needs an inverse, so max is a configuration error. */
int oracle_sat_included(const void *in, void *out, int dtype, int op, int d,
                        const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    set_threads(nthreads);
    if (dtype == 0 && op == 0) return sat_included_f32_add(in, out, d, ext, k);
    if (dtype == 1 && op == 0) return sat_included_f64_add(in, out, d, ext, k);
    if (dtype == 2 && op == 0) return sat_included_i64_add(in, out, d, ext, k);
    if (dtype == 2 && op == 2) return sat_included_i64_mod(in, out, d, ext, k);
    return ORC_CONFIG;
}

/* "satc" (excluded.py:83-85): fold(A) (-) sat_included(A), like bdbsc. */
int oracle_satc_excluded(const void *in, void *out, int dtype, int op, int d,
                         const int64_t *ext, const int64_t *box, int nthreads) {
    int rc = oracle_sat_included(in, out, dtype, op, d, ext, box, nthreads);
    if (rc) return rc;
    int64_t N = prod_range(ext, 0, d);
    if (dtype == 0) {
        float total = fold_f32_add(in, N);
        float *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = total - o[i];
    } else if (dtype == 1) {
        double total = fold_f64_add(in, N);
        double *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = total - o[i];
    } else if (op == 0) {
        int64_t total = fold_i64_add(in, N);
        int64_t *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = i64_sub(total, o[i]);
    } else {
        int64_t total = floor_mod(fold_i64_add(in, N));
        int64_t *o = out;
        for (int64_t i = 0; i < N; ++i) o[i] = mod_sub(total, o[i]);
    }
    return ORC_OK;
}

int oracle_brute_included(const void *in, void *out, int dtype, int op, int d,
                          const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    set_threads(nthreads);
    DISPATCH(brute_inc, in, out, d, ext, k);
    return ORC_OK;
}

int oracle_brute_excluded(const void *in, void *out, int dtype, int op, int d,
                          const int64_t *ext, const int64_t *box, int nthreads) {
    int64_t k[16];
    int rc = normalize(d, ext, box, k);
    if (rc) return rc;
    set_threads(nthreads);
    DISPATCH(brute_exc, in, out, d, ext, k);
    return ORC_OK;
}

/* Sequential fold in the data type (MonoidOps.fold), exposed for tests. */
int oracle_fold(const void *in, int64_t n, int dtype, int op, void *result) {
    if (dtype == 0 && op == 0) { *(float *)result = fold_f32_add(in, n); return ORC_OK; }
    if (dtype == 1 && op == 0) { *(double *)result = fold_f64_add(in, n); return ORC_OK; }
    if (dtype == 2 && op == 0) { *(int64_t *)result = fold_i64_add(in, n); return ORC_OK; }
    if (dtype == 2 && op == 1) { *(int64_t *)result = fold_i64_max(in, n); return ORC_OK; }
    if (dtype == 2 && op == 2) { *(int64_t *)result = floor_mod(fold_i64_add(in, n)); return ORC_OK; }
    return ORC_CONFIG;
}
