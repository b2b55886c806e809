"""The hot-path entry points, with the reference's signatures.

=============================  ==========================================
this module                    reference (pkg/src/exsum)
=============================  ==========================================
bdbs_included(t, box)          included.py:124-129
bdbs_excluded(t, box)          excluded.py:88-90 (+ _complement :72-75)
box_complement_excluded(t,box) excluded.py:129-159
sat_included(t, box)           included.py:98-121 (+ sat_build :37-42)
sat_excluded(t, box)           excluded.py:83-85
corners_excluded(t, box, c)    excluded.py:200-225 (2-D, 3-D)
corners_spine_excluded(t,b,c)  excluded.py:228-262 (2-D, 3-D)
bdbs_1d(ops, values, k)        scan.py:53-58
windowed_sum_axis(ops,v,k,ax)  scan.py:61-102 (in place on ``v``)
ALGORITHMS / AlgorithmInfo     bench.py:45-100 (the plug-in registry)
=============================  ==========================================

Every call validates exactly like the reference (``normalize_box``; a weak
route on a monoid without inverse raises ``ConfigurationError`` before any
work, like bench.check_algorithm_config) and then runs on the B200 through
the C ABI.  Data placement decides the path:

* ``t.data`` is a CUDA ``torch.Tensor``: device pointers go straight to the
  stream-ordered entry points on ``torch.cuda.current_stream()``; the result is
  a new CUDA tensor (no host copies).
* ``t.data`` is a numpy array (the reference's own Tensor, for instance):
  ``exsum_run_host`` copies it to HBM, computes, and copies the result back.

The result is a new tensor carrying the caller's ``t.ops`` (bench.py:221,233
re-wraps results with ``with_ops``), of the caller's Tensor class.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigurationError, UsageError
from .monoid import device_operator, modulus_of
from .tensor import Tensor, is_torch, normalize_box, np_dtype_of

_DT_NAME = {np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
            np.dtype(np.int64): "int64"}


_NEEDS_INVERSE = ("bdbsc", "sat", "satc")  # bench.py:60-76 needs_inverse


def _prepare(t, box, route):
    dtype, op, has_inverse = device_operator(t.ops)
    if route in _NEEDS_INVERSE and not has_inverse:
        raise ConfigurationError(
            f"algorithm {route!r} requires an invertible monoid, but {t.ops.name!r} has no inverse"
        )
    data = t.data
    ext = tuple(int(v) for v in data.shape)
    k = normalize_box(ext, box)
    if np_dtype_of(data) != dtype:
        raise UsageError(f"dtype {np_dtype_of(data)} does not match monoid {t.ops.name}")
    return _DT_NAME[dtype], op, ext, k, modulus_of(t.ops)


def _rewrap(t, out):
    try:
        return type(t)(t.ops, out)
    except Exception:
        return Tensor(t.ops, out)


# per-call constants of a (route, dtype, op, extents, box, modulus) combination:
# the workspace size and the ctypes argument arrays (small calls are host-bound)
_PLAN_CACHE: dict = {}
# one growing workspace per (device, stream): work on a stream is ordered, so a
# call may reuse the buffer the previous call on the same stream used
_WS_CACHE: dict = {}


def _plan(route, dtype, op, ext, k, modulus):
    key = (route, dtype, op, ext, k, modulus)
    p = _PLAN_CACHE.get(key)
    if p is None:
        p = (_native.workspace_bytes(route, dtype, op, ext, k, modulus),
             _native.i64_array(ext), _native.i64_array(k))
        if len(_PLAN_CACHE) > 4096:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = p
    return p


def _workspace(device, stream, nbytes):
    import torch

    key = (device.index, stream)
    ws = _WS_CACHE.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = ws
    return ws


def release_workspace_cache() -> None:
    """Drop the cached per-stream workspaces (and the library's host-path buffers)."""
    _WS_CACHE.clear()
    _native.load().exsum_release_cache()


def run_device(route: str, x, dtype: str, op: str, ext, k, out=None, modulus: int = 0):
    """Run ``route`` on a CUDA torch tensor; returns the output tensor.
    ``modulus``: m of a ``mod-add:<m>`` operator (op == "mod-add")."""
    import torch

    if not x.is_cuda:
        raise UsageError("run_device needs a CUDA tensor")
    x = x.contiguous()
    if x.data_ptr() % 16:
        x = x.clone()  # a view off 16-byte alignment: the fused kernels need aligned rows
    if out is None:
        out = torch.empty_like(x)
    elif out.data_ptr() % 16 or not out.is_contiguous():
        raise UsageError("out must be a contiguous, 16-byte aligned CUDA tensor")
    L = _native.load()
    ext, k = tuple(ext), tuple(k)
    ws_bytes, c_ext, c_k = _plan(route, dtype, op, ext, k, int(modulus))
    with torch.cuda.device(x.device):
        stream = torch.cuda.current_stream(x.device).cuda_stream
        ws = _workspace(x.device, stream, ws_bytes)
        _native.check(L.exsum_route(_native.ROUTE[route], x.data_ptr(), out.data_ptr(),
                                    _native.DTYPE[dtype], _native.OP[op], int(modulus), len(ext),
                                    c_ext, c_k, ws.data_ptr(), ws_bytes, stream))
    return out


def run_host(route: str, a: np.ndarray, dtype: str, op: str, ext, k, out=None,
             modulus: int = 0) -> np.ndarray:
    """Run ``route`` on a host array through exsum_run_host (H2D, compute, D2H).

    ``out`` (optional) receives the result; pass page-locked buffers (e.g. a
    numpy view of a pinned torch tensor) for full PCIe bandwidth."""
    a = np.ascontiguousarray(a)
    if out is None:
        out = np.empty_like(a)
    elif out.shape != a.shape or out.dtype != a.dtype or not out.flags.c_contiguous:
        raise UsageError("out must be a C-contiguous array of the input's shape and dtype")
    L = _native.load()
    _native.check(L.exsum_route_host(_native.ROUTE[route], a.ctypes.data, out.ctypes.data,
                                     _native.DTYPE[dtype], _native.OP[op], int(modulus), len(ext),
                                     _native.i64_array(ext), _native.i64_array(k)))
    return out


def run_host_batch(route: str, arrays, dtype: str, op: str, ext, k, outs=None,
                   modulus: int = 0):
    """Run ``route`` over a list of same-shaped host arrays with the copies of
    consecutive arrays overlapped (exsum_route_host_batch); returns the outputs."""
    import ctypes

    arrays = [np.ascontiguousarray(a) for a in arrays]
    if outs is None:
        outs = [np.empty_like(a) for a in arrays]
    for a, o in zip(arrays, outs):
        if a.shape != tuple(ext) or o.shape != a.shape or o.dtype != a.dtype or \
                not o.flags.c_contiguous:
            raise UsageError("every input and output must have the batch's extents and dtype")
    L = _native.load()
    n = len(arrays)
    pin = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrays])
    pout = (ctypes.c_void_p * n)(*[o.ctypes.data for o in outs])
    _native.check(L.exsum_route_host_batch(_native.ROUTE[route], n, pin, pout,
                                           _native.DTYPE[dtype], _native.OP[op], int(modulus),
                                           len(ext), _native.i64_array(ext), _native.i64_array(k)))
    return outs


def run_many(algo: str, tensors, box):
    """One registry entry over many same-shaped tensors (AlgorithmInfo.run per
    tensor), returning the result tensors in order.  Host (numpy) tensors go
    through exsum_route_host_batch, which overlaps the host->device copy of the
    next array with the device->host copy of the previous one; device tensors
    run back to back on the current stream."""
    tensors = list(tensors)
    if not tensors:
        return []
    if algo in ("corners", "corners-spine"):
        return [ALGORITHMS[algo].run(t, box) for t in tensors]
    resolve_algorithm(algo)
    prepared = [_prepare(t, box, algo) for t in tensors]
    if len({(p[0], p[1], p[2], p[3], p[4]) for p in prepared}) != 1:
        raise UsageError("run_many needs tensors of one shape, dtype and monoid")
    dtype, op, ext, k, m = prepared[0]
    if any(is_torch(t.data) for t in tensors):
        return [ALGORITHMS[algo].run(t, box) for t in tensors]
    outs = run_host_batch(algo, [np.asarray(t.data) for t in tensors], dtype, op, ext, k,
                          modulus=m)
    return [_rewrap(t, o) for t, o in zip(tensors, outs)]


def _route(route, t, box):
    dtype, op, ext, k, m = _prepare(t, box, route)
    data = t.data
    if is_torch(data):
        if data.is_cuda:
            return _rewrap(t, run_device(route, data, dtype, op, ext, k, modulus=m))
        out = run_host(route, data.numpy(), dtype, op, ext, k, modulus=m)
        import torch

        return _rewrap(t, torch.from_numpy(out))
    return _rewrap(t, run_host(route, np.asarray(data), dtype, op, ext, k, modulus=m))


def bdbs_included(t, box):
    """Strong included sum: out[x] = (+) over the clipped box [x, x+k)."""
    return _route("bdbs", t, box)


def bdbs_excluded(t, box):
    """Weak excluded sum: total (-) included (needs an invertible monoid)."""
    return _route("bdbsc", t, box)


def box_complement_excluded(t, box):
    """Strong excluded sum over the complement of the clipped box (any monoid)."""
    return _route("box-complement", t, box)


def sat_included(t, box):
    """Included sum through a running-sum table and 2^d corner queries
    (needs an invertible monoid)."""
    return _route("sat", t, box)


def sat_excluded(t, box):
    """Total minus the table-based included sum (needs an invertible monoid)."""
    return _route("satc", t, box)


def _corner_checks(t, box, c, label):
    """_corner_rules (excluded.py:191-197) then normalize_box then the space
    factor, in the reference's order."""
    d = len(t.data.shape)
    if d not in (2, 3):
        raise ConfigurationError(
            f"corner decomposition is only defined for 2-D and 3-D tensors, got {d}-D"
        )
    normalize_box(tuple(int(v) for v in t.data.shape), box)
    if not isinstance(c, (int, np.integer)) or not 1 <= int(c) <= d:
        raise UsageError(f"{label} must be in [1, {d}] for a {d}-D tensor, got {c}")


def corners_excluded(t, box, buffers: int = 1):
    """Strong excluded sum by the 2^d corner decomposition (any monoid, 2-D/3-D).
    ``buffers`` is the reference's space factor; the GPU keeps one scanned
    copy whatever its value (the values do not depend on it)."""
    _corner_checks(t, box, buffers, "corners buffer count")
    return _route("corners", t, box)


def corners_spine_excluded(t, box, cache_depth: int = 1):
    """Spine-cached corner decomposition (same values as corners_excluded)."""
    _corner_checks(t, box, cache_depth, "cache depth")
    return _route("corners-spine", t, box)


def bdbs_1d(ops, values, k):
    """Windowed sums of a 1-D sequence: out[x] = fold(values[x : x+k])."""
    dtype, op, _ = device_operator(ops)
    arr = np.array(values, dtype=dtype).reshape(-1)
    (kk,) = normalize_box(arr.shape, (k,))
    return run_host("bdbs", arr, _DT_NAME[dtype], op, arr.shape, (kk,), modulus=modulus_of(ops))


def windowed_sum_axis(ops, view, k, axis):
    """In-place windowed sums along ``axis`` of ``view`` (scan.py:61-102)."""
    dtype, op, _ = device_operator(ops)
    ext = tuple(int(v) for v in view.shape)
    if not 0 <= axis < len(ext):
        raise UsageError(f"axis {axis} out of range for {len(ext)}-D view")
    if int(k) < 1:
        raise UsageError(f"every box side must be >= 1, got {k}")
    if min(ext, default=1) == 0 or int(k) == 1:
        return
    box = tuple(int(k) if i == axis else 1 for i in range(len(ext)))
    t = Tensor(_OpsShim(ops), view.contiguous() if is_torch(view) else np.ascontiguousarray(view))
    res = bdbs_included(t, box)
    if is_torch(view):
        view.copy_(res.data)
    else:
        view[...] = res.data


class _OpsShim:
    def __init__(self, ops):
        self.inner = ops
        self.name = getattr(ops, "name", "?")
        self.dtype = ops.dtype
        self.identity = getattr(ops, "identity", 0)


# -- the plug-in registry (bench.py:45-100) -------------------------------------


@dataclass(frozen=True)
class AlgorithmInfo:
    name: str
    fn: object
    kind: str  # "included" or "excluded"
    needs_inverse: bool
    dims: object = None
    cache_arg: str = ""

    def run(self, t, box, cache: int = 1):
        if self.cache_arg:
            return self.fn(t, box, **{self.cache_arg: cache})
        return self.fn(t, box)


ALGORITHMS = {
    info.name: info
    for info in (
        AlgorithmInfo("sat", sat_included, "included", True),
        AlgorithmInfo("bdbs", bdbs_included, "included", False),
        AlgorithmInfo("satc", sat_excluded, "excluded", True),
        AlgorithmInfo("bdbsc", bdbs_excluded, "excluded", True),
        AlgorithmInfo("box-complement", box_complement_excluded, "excluded", False),
        AlgorithmInfo("corners", corners_excluded, "excluded", False, {2, 3}, "buffers"),
        AlgorithmInfo("corners-spine", corners_spine_excluded, "excluded", False, {2, 3},
                      "cache_depth"),
    )
}


def resolve_algorithm(name: str) -> AlgorithmInfo:
    info = ALGORITHMS.get(name)
    if info is None:
        raise ConfigurationError(
            f"unknown algorithm {name!r}; choose from {', '.join(sorted(ALGORITHMS))}"
        )
    return info


def check_algorithm_config(info: AlgorithmInfo, ops, d=None) -> None:
    """Reject impossible algorithm/monoid combinations before any work (bench.py:88-100)."""
    _, _, has_inverse = device_operator(ops)
    if info.needs_inverse and not has_inverse:
        raise ConfigurationError(
            f"algorithm {info.name!r} requires an invertible monoid, "
            f"but {getattr(ops, 'name', ops)!r} has no inverse"
        )
    if d is not None and info.dims is not None and d not in info.dims:
        dims = ", ".join(str(v) for v in sorted(info.dims))
        raise ConfigurationError(
            f"algorithm {info.name!r} supports {dims}-D tensors only, got {d}-D"
        )


def register_with_reference(bench_module) -> None:
    """Swap the reference's registry entries for the B200 routes.

    ``bench_module`` is the reference's ``exsum.bench``; afterwards
    ``exsum run --algo sat|bdbs|satc|bdbsc|box-complement|corners|corners-spine``
    executes on the GPU
    (the monkeypatch precedent is test_bench.py:243-245).
    """
    ref_info = bench_module.AlgorithmInfo
    for name, info in ALGORITHMS.items():
        bench_module.ALGORITHMS[name] = ref_info(name, info.fn, info.kind, info.needs_inverse,
                                                 info.dims, info.cache_arg)
