"""The reference's building blocks, on the GPU.

=====================================  =========================================
this module                            reference (pkg/src/exsum)
=====================================  =========================================
reduced_slice(t, dim)                  scan.py:105-110 (a view, no work)
prefix_along_dim(t, dim)               scan.py:113-115
suffix_along_dim(t, dim)               scan.py:118-120
bdbs_along_dim(t, box, dim, scan_dim)  scan.py:123-129
add_contribution(src, dst, dim, off)   excluded.py:111-126
accumulate(ops, arr, axis, reverse)    MonoidOps.accumulate  monoid.py:156-159, 196-198,
                                       224-226, 280-283
combine_into / rcombine_into /         MonoidOps bulk kernels monoid.py:145-155, 184-195,
subtract_into / rsubtract_scalar       219-223, 268-279
fold(ops, arr)                         MonoidOps.fold  monoid.py:161-164, 200-204, 229-232,
                                       284-286
=====================================  =========================================

The monoids of this package expose the same bulk methods (``ops.combine_into(dst,
src)``, ``ops.accumulate(arr, axis)``, ``ops.fold(arr)`` ...), which call these.

Arrays are modified in place, like the reference.  A CUDA ``torch.Tensor`` is
worked on where it lives; a numpy array (or view) is copied to the device, the
kernel runs there, and the result is written back into it -- the arithmetic
always runs in the CUDA kernels of ``libexsum_b200.so`` (no CPU fallback).
Sequential scans keep numpy's association, so float ``accumulate`` results are
bit-identical to numpy's; ``fold`` is a deterministic tree (float32 accumulates
in float64), which differs from numpy's sequential float fold by reassociation.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import ConfigurationError, UsageError
from .monoid import device_operator, modulus_of
from .tensor import is_torch, normalize_box

_DT_NAME = {np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
            np.dtype(np.int64): "int64"}


def _codes(ops, dtype):
    want, op, has_inverse = device_operator(ops)
    if np.dtype(dtype) != want:
        raise UsageError(f"dtype {np.dtype(dtype)} does not match monoid {getattr(ops, 'name', ops)}")
    return _native.DTYPE[_DT_NAME[want]], _native.OP[op], modulus_of(ops), has_inverse


class _OnDevice:
    """A contiguous CUDA tensor holding `arr`, written back on exit when `arr`
    is not that tensor itself (numpy arrays, views, non-contiguous tensors)."""

    def __init__(self, arr, write_back=True):
        import torch

        self.arr = arr
        self.write_back = write_back
        if is_torch(arr) and arr.is_cuda and arr.is_contiguous():
            self.dev, self.own = arr, True
        elif is_torch(arr):
            self.dev, self.own = arr.detach().contiguous().cuda(), False
        else:
            self.dev = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
            self.own = False

    def __enter__(self):
        return self.dev

    def __exit__(self, *exc):
        if exc[0] is None and not self.own and self.write_back:
            if is_torch(self.arr):
                self.arr.copy_(self.dev)
            else:
                self.arr[...] = self.dev.cpu().numpy()
        return False


def _stream(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream


def _dtype_of(arr):
    if is_torch(arr):
        import torch

        return {torch.float32: np.float32, torch.float64: np.float64,
                torch.int64: np.int64}.get(arr.dtype, np.dtype("V1"))
    return np.asarray(arr).dtype


# -- MonoidOps bulk kernels ------------------------------------------------------


def accumulate(ops, arr, axis: int, reverse: bool = False) -> None:
    """Running fold along `axis`, in place (reversed: a suffix fold)."""
    dt, op, m, _ = _codes(ops, _dtype_of(arr))
    shape = tuple(int(v) for v in arr.shape)
    if not shape or min(shape) == 0:
        return
    axis = int(axis) % len(shape)
    L = _native.load()
    with _OnDevice(arr) as x:
        import torch

        need = ctypes.c_size_t(0)
        _native.check(L.exsum_scan_workspace_bytes(dt, op, m, len(shape), _native.i64_array(shape),
                                                   axis, ctypes.byref(need)))
        ws = torch.empty(max(int(need.value), 1), dtype=torch.uint8, device=x.device)
        _native.check(L.exsum_scan_axis(x.data_ptr(), x.data_ptr(), dt, op, m, len(shape),
                                        _native.i64_array(shape), axis, 1 if reverse else 0,
                                        ws.data_ptr(), int(need.value), _stream(x)))


def _elementwise(ops, dst, src, scalar, kind):
    dt, op, m, has_inverse = _codes(ops, _dtype_of(dst))
    if kind > 0 and not has_inverse:
        raise ConfigurationError(f"monoid {ops.name!r} has no inverse")
    if src is not None and tuple(src.shape) != tuple(dst.shape):
        raise UsageError(f"shape mismatch {tuple(src.shape)} vs {tuple(dst.shape)}")
    n = int(np.prod(dst.shape)) if dst.shape else 1
    if n == 0:
        return
    L = _native.load()
    with _OnDevice(dst) as d:
        sptr = None
        keep = None
        if src is not None:
            if _dtype_of(src) != _dtype_of(dst):
                raise UsageError("dst and src must share a dtype")
            keep = _OnDevice(src, write_back=False).dev
            sptr = keep.data_ptr()
        sc = None
        if scalar is not None:
            sc = np.array([scalar], dtype=_dtype_of(dst))
        _native.check(L.exsum_elementwise(d.data_ptr(), sptr,
                                          None if sc is None else sc.ctypes.data, dt, op, m, kind,
                                          n, _stream(d)))
        if sc is not None or keep is not None:
            import torch

            torch.cuda.current_stream(d.device).synchronize()  # host scalar / staged src lifetime


def combine_into(ops, dst, src) -> None:
    """dst = dst (+) src, elementwise, in place."""
    _elementwise(ops, dst, src, None, 0)


def rcombine_into(ops, dst, src) -> None:
    """dst = src (+) dst (every operator here is commutative: same as combine_into)."""
    _elementwise(ops, dst, src, None, 0)


def subtract_into(ops, dst, src) -> None:
    """dst = dst (-) src (invertible monoids)."""
    _elementwise(ops, dst, src, None, 1)


def rsubtract_scalar(ops, total, dst) -> None:
    """dst = total (-) dst (invertible monoids; excluded.py:72-75)."""
    _elementwise(ops, dst, None, total, 2)


def fold(ops, arr):
    """Fold of every element (the identity for an empty array), as a Python scalar."""
    dt, op, m, _ = _codes(ops, _dtype_of(arr))
    n = int(np.prod(arr.shape)) if arr.shape else 1
    L = _native.load()
    import torch

    with _OnDevice(arr, write_back=False) as x:
        res = torch.zeros(1, dtype=x.dtype, device=x.device)
        nb = int(L.exsum_fold_workspace_bytes())
        ws = torch.empty(nb, dtype=torch.uint8, device=x.device)
        _native.check(L.exsum_fold(x.data_ptr(), res.data_ptr(), dt, op, m, n, ws.data_ptr(), nb,
                                   _stream(x)))
        return res.item()


# -- the excluded-sum pipeline's helpers (scan.py:105-129, excluded.py:111-126) --


def reduced_slice(t, dim: int):
    """View of t with every dimension before `dim` pinned at its last index."""
    nd = len(t.data.shape)
    if not 0 <= dim < nd:
        raise UsageError(f"dimension {dim} out of range for {nd}-D tensor")
    return t.data[tuple(int(n) - 1 for n in t.data.shape[:dim])]


def prefix_along_dim(t, dim: int) -> None:
    """Prefix scan along `dim` on the reduced slice, in place."""
    accumulate(t.ops, reduced_slice(t, dim), 0)


def suffix_along_dim(t, dim: int) -> None:
    """Suffix scan along `dim` on the reduced slice, in place."""
    accumulate(t.ops, reduced_slice(t, dim), 0, reverse=True)


def bdbs_along_dim(t, box, dim: int, scan_dim: int) -> None:
    """Windowed sums along `scan_dim` on the reduced slice at `dim`, in place."""
    from .routes import windowed_sum_axis

    k = normalize_box(tuple(int(v) for v in t.data.shape), box)
    if scan_dim < dim:
        raise UsageError(f"scan dimension {scan_dim} precedes reduced dimension {dim}")
    windowed_sum_axis(t.ops, reduced_slice(t, dim), k[scan_dim], scan_dim - dim)


def add_contribution(src, dst, dim: int, offset: int) -> None:
    """dst[.., x_dim, ..] (+)= src_reduced[x_dim + offset, ..] wherever in range,
    broadcast over the dims before `dim` (accumulates)."""
    shape = tuple(int(v) for v in dst.data.shape)
    if tuple(int(v) for v in src.data.shape) != shape:
        raise UsageError("add_contribution needs tensors of equal extents")
    if not 0 <= dim < len(shape):
        raise UsageError(f"dimension {dim} out of range for {len(shape)}-D tensor")
    dt, op, m, _ = _codes(dst.ops, _dtype_of(dst.data))
    L = _native.load()
    with _OnDevice(dst.data) as d:
        s = _OnDevice(reduced_slice(src, dim), write_back=False).dev
        _native.check(L.exsum_add_contribution(s.data_ptr(), d.data_ptr(), dt, op, m, len(shape),
                                               _native.i64_array(shape), int(dim), int(offset),
                                               _stream(d)))
        import torch

        torch.cuda.current_stream(d.device).synchronize()  # staged src lifetime


__all__ = ["accumulate", "add_contribution", "bdbs_along_dim", "combine_into", "fold",
           "prefix_along_dim", "rcombine_into", "reduced_slice", "rsubtract_scalar",
           "subtract_into", "suffix_along_dim"]
