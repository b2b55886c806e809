"""Parity helpers shared by the GPU tests and bench.py (test infrastructure).

Exactness contract (north star):
  * int64 + and max: bit-exact, every route.
  * float BDBS: bit-exact -- the kernels keep the reference's association
    (in-block right-nested suffix, left-nested prefix, axes in order).
  * float BDBSC and box-complement: |got - want| <= tau * S(x), where want is
    the reference algorithm evaluated in float64 (the CPU oracle on the
    float64-upcast input), S(x) is a magnitude bound of every partial sum that
    feeds x, and tau = D * u with u the unit roundoff of the data type and D
    a bound on the number of roundings on any path to x:
      - BDBSC: S(x) = sum(|A|) (the total dominates), D = sum_i(2 k_i) + 8;
      - box-complement: S(x) = box_complement(|A|)(x), the same route applied
        to |A|.  The route is strong: every term feeding x is a
        partial sum of |A| over a subset of x's complement (no subtraction
        anywhere, excluded.py:130), so an inverse-free evaluation's error is
        bounded by D * u * S(x) with D = sum_i(n_i + 2 k_i) + 16 (full-axis
        scans are the longest chains).  A weak evaluation (row total minus
        window) would not meet it where x's box holds large mass.
      - sat / satc: every table entry is a prefix sum bounded by
        sum(|A|) and the query folds 2^d of them, so S(x) = 2^d * sum(|A|)
        (+ sum(|A|) for satc's total) and D = sum_i(n_i) + 2^d + 8.  Where the
        scans run unsegmented the float tables are bit-identical to the
        reference's (numpy's sequential accumulate), and so is sat itself.
    Both sides round: tau * S(x) = (D_gpu * u + D_ref * 2^-53) * S(x), the
    oracle always running in float64 (tau = (D_gpu + D_ref) u).
    D_ref follows the reference's own association: BDBS sum_i(2 k_i - 1),
    BDBSC N + sum_i(2 k_i) (its total is one sequential fold over all N
    elements, monoid.py:200-204), box-complement sum_i(n_i - 1) + sum_i(2 k_i)
    + 2d.  Next to float32's u = 2^-24 the oracle's share is negligible
    except for BDBSC's sequential total; for float64 data it matters.
"""

from __future__ import annotations

import numpy as np

U = {np.dtype(np.float32): 2.0**-24, np.dtype(np.float64): 2.0**-53}


def depth(route, ext, k):
    if route == "bdbs":
        return sum(2 * kk for kk in k) + 4
    if route == "bdbsc":
        return sum(2 * kk for kk in k) + 8
    if route in ("sat", "satc"):
        return sum(ext) + 2 ** len(ext) + 8
    return sum(n + 2 * kk for n, kk in zip(ext, k)) + 16


def depth_ref(route, ext, k):
    """Rounding depth of the reference's own association."""
    if route == "bdbs":
        return sum(2 * kk - 1 for kk in k)
    if route == "bdbsc":
        return int(np.prod(ext)) + sum(2 * kk for kk in k)
    if route in ("sat", "satc"):
        return depth(route, ext, k)
    return sum(n - 1 for n in ext) + sum(2 * kk for kk in k) + 2 * len(ext)


def float_tolerance(route, a, k, oracle_mod):
    """Elementwise tolerance array for a float route (see module docstring)."""
    ext = a.shape
    a64 = np.abs(a.astype(np.float64))
    tau = depth(route, ext, k) * U[np.dtype(a.dtype)] + depth_ref(route, ext, k) * 2.0**-53
    if route == "bdbsc":
        S = np.full(ext, a64.sum())
    elif route in ("sat", "satc"):
        S = np.full(ext, (2 ** len(ext) + (route == "satc")) * a64.sum())
    elif route == "box-complement":
        S = oracle_mod.box_complement_excluded(a64, k)
    else:
        S = oracle_mod.bdbs_included(a64, k)
    return tau * S + np.finfo(np.float64).tiny


def compare(route, got, want, a, k, oracle_mod):
    """Return (ok, max_err_over_tol, max_rel_err) per the exactness contract."""
    got = np.asarray(got)
    want = np.asarray(want)
    if got.shape != want.shape:
        return False, float("inf"), float("inf")
    if got.dtype.kind != "f" or route == "bdbs":
        ok = np.array_equal(got.view(np.uint8), want.astype(got.dtype).view(np.uint8))
        return ok, 0.0 if ok else float("inf"), 0.0 if ok else float("inf")
    tol = float_tolerance(route, a, k, oracle_mod)
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    ratio = float(np.max(err / tol)) if err.size else 0.0
    rel = float(np.max(err / np.maximum(np.abs(want.astype(np.float64)), 1e-300))) if err.size else 0.0
    return ratio <= 1.0, ratio, rel


def float64_oracle(route, a, box, oracle_mod, op="add"):
    """Reference algorithm evaluated in float64 on the upcast input."""
    if a.dtype.kind == "f":
        return oracle_mod.ROUTES[route](a.astype(np.float64), box, op)
    return oracle_mod.ROUTES[route](a, box, op)
