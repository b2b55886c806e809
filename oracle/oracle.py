"""CPU oracle for the box-sum hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / the timed CPU baseline.  The product package
(``paper_2106_00124_b200``) never imports it and has no CPU fallback.

Two tiers, both pinned to the reference (``/root/reference/pkg``) by
``tests/test_oracle.py`` against golden vectors produced by running the
reference itself (``tests/golden/make_golden.py``):

* ``liboracle.so`` (``exsum_oracle.c``): a C restatement of
  ``windowed_sum_axis`` (scan.py:61-102), ``bdbs_included`` (included.py:124-129),
  ``bdbs_excluded`` (excluded.py:72-75,88-90) and ``box_complement_excluded``
  (excluded.py:129-159) with the reference's exact floating-point association,
  so it is bit-identical to the reference for every dtype.
* ``sat_included`` / ``sat_excluded`` (included.py:37-121, excluded.py:83-85) and the
  ``mod-add:<m>`` monoid (monoid.py:235-286) for every route (``op="mod-add:<m>"``).
* ``brute_included`` / ``brute_excluded``: restatements of the brute-force
  ``oracle_included`` / ``oracle_excluded`` (oracle.py:37-71), in C for speed and
  in pure Python (``py_brute_*``) for tiny cases.
"""

from __future__ import annotations

import ctypes
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

DTYPE_CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int64): 2}
OP_CODES = {"add": 0, "max": 1, "mod-add": 2}
IDENTITY = {
    ("add", np.dtype(np.float32)): np.float32(0.0),
    ("add", np.dtype(np.float64)): np.float64(0.0),
    ("add", np.dtype(np.int64)): np.int64(0),
    ("max", np.dtype(np.int64)): np.int64(np.iinfo(np.int64).min),
}

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        for name in (
            "oracle_bdbs_included",
            "oracle_bdbsc_excluded",
            "oracle_box_complement_excluded",
            "oracle_sat_included",
            "oracle_satc_excluded",
            "oracle_corners_excluded",
            "oracle_brute_included",
            "oracle_brute_excluded",
        ):
            fn = getattr(L, name)
            fn.argtypes = [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                i64p, i64p, ctypes.c_int,
            ]
            fn.restype = ctypes.c_int
        L.oracle_windowed_pass.argtypes = [
            ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, ctypes.c_int,
            ctypes.c_int64, ctypes.c_int,
        ]
        L.oracle_windowed_pass.restype = ctypes.c_int
        L.oracle_fold.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
        ]
        L.oracle_fold.restype = ctypes.c_int
        L.oracle_set_modulus.argtypes = [ctypes.c_int64]
        L.oracle_set_modulus.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _codes(arr: np.ndarray, op: str):
    """op: "add", "max" or "mod-add:<m>" (sets the oracle's modulus)."""
    dt = DTYPE_CODES.get(arr.dtype)
    base, _, mod = op.partition(":")
    if dt is None or base not in OP_CODES or (base == "mod-add") != bool(mod):
        raise OracleError(f"unsupported dtype/op {arr.dtype}/{op}")
    if base == "mod-add":
        if lib().oracle_set_modulus(int(mod)) != 0:
            raise OracleError(f"bad modulus {mod}")
    return dt, OP_CODES[base]


def _i64(seq):
    a = (ctypes.c_int64 * len(seq))(*[int(v) for v in seq])
    return a


def _run(fn_name: str, a: np.ndarray, box, op: str, nthreads: int) -> np.ndarray:
    a = np.ascontiguousarray(a)
    out = np.empty_like(a)
    dt, opc = _codes(a, op)
    fn = getattr(lib(), fn_name)
    rc = fn(
        a.ctypes.data, out.ctypes.data, dt, opc, a.ndim, _i64(a.shape), _i64(box), int(nthreads)
    )
    if rc != 0:
        raise OracleError(f"{fn_name} returned {rc}")
    return out


def bdbs_included(a, box, op="add", nthreads=0):
    return _run("oracle_bdbs_included", a, box, op, nthreads)


def bdbs_excluded(a, box, op="add", nthreads=0):
    return _run("oracle_bdbsc_excluded", a, box, op, nthreads)


def box_complement_excluded(a, box, op="add", nthreads=0):
    return _run("oracle_box_complement_excluded", a, box, op, nthreads)


def sat_included(a, box, op="add", nthreads=0):
    return _run("oracle_sat_included", a, box, op, nthreads)


def sat_excluded(a, box, op="add", nthreads=0):
    return _run("oracle_satc_excluded", a, box, op, nthreads)


def corners_excluded(a, box, op="add", nthreads=0):
    return _run("oracle_corners_excluded", a, box, op, nthreads)


def brute_included(a, box, op="add", nthreads=0):
    return _run("oracle_brute_included", a, box, op, nthreads)


def brute_excluded(a, box, op="add", nthreads=0):
    return _run("oracle_brute_excluded", a, box, op, nthreads)


ROUTES = {
    "bdbs": bdbs_included,
    "bdbsc": bdbs_excluded,
    "box-complement": box_complement_excluded,
    "sat": sat_included,
    "satc": sat_excluded,
    "corners": corners_excluded,
    "corners-spine": corners_excluded,
}


def windowed_pass(a, axis, k, op="add", nthreads=0):
    a = np.array(a, copy=True, order="C")
    dt, opc = _codes(a, op)
    rc = lib().oracle_windowed_pass(
        a.ctypes.data, dt, opc, a.ndim, _i64(a.shape), int(axis), int(k), int(nthreads)
    )
    if rc != 0:
        raise OracleError(f"oracle_windowed_pass returned {rc}")
    return a


def fold(a, op="add"):
    a = np.ascontiguousarray(a)
    dt, opc = _codes(a, op)
    res = np.zeros(1, dtype=a.dtype)
    rc = lib().oracle_fold(a.ctypes.data, a.size, dt, opc, res.ctypes.data)
    if rc != 0:
        raise OracleError(f"oracle_fold returned {rc}")
    return res[0]


# -- pure-Python brute force (oracle.py:22-71 restated; tiny cases only) -------


def _combine(op):
    if op == "add":
        return lambda a, b: a + b
    if op.startswith("mod-add:"):
        m = int(op.split(":")[1])
        return lambda a, b: (int(a) + int(b)) % m
    return lambda a, b: a if a >= b else b


def py_brute_included(extents, flat, box, op, identity):
    combine = _combine(op)
    strides = [1] * len(extents)
    for i in range(len(extents) - 2, -1, -1):
        strides[i] = strides[i + 1] * extents[i + 1]
    out = []
    for x in itertools.product(*[range(n) for n in extents]):
        acc = None
        for y in itertools.product(*[range(xi, min(xi + ki, ni)) for xi, ki, ni in zip(x, box, extents)]):
            v = flat[sum(a * b for a, b in zip(y, strides))]
            acc = v if acc is None else combine(acc, v)
        out.append(identity if acc is None else acc)
    return out


def py_brute_excluded(extents, flat, box, op, identity):
    combine = _combine(op)
    out = []
    for x in itertools.product(*[range(n) for n in extents]):
        acc = None
        for idx, y in enumerate(itertools.product(*[range(n) for n in extents])):
            if not all(xi <= yi < xi + ki for xi, yi, ki in zip(x, y, box)):
                v = flat[idx]
                acc = v if acc is None else combine(acc, v)
        out.append(identity if acc is None else acc)
    return out
