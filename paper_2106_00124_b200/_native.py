"""ctypes binding of libexsum_b200.so (the C ABI in include/exsum_b200.h).

This is the binding a maintainer of the reference would add:
the reference is pure Python, so its FFI for a native path is ctypes.  The
library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  If it
is missing, every entry point raises ``DeviceError`` -- there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigurationError, DeviceError, UsageError

# EXSUM_LIB overrides the library (ablation builds in measurements); the
# default is the in-tree build.
LIB_PATH = os.environ.get("EXSUM_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libexsum_b200.so")

DTYPE = {"float32": 0, "float64": 1, "int64": 2}
OP = {"add": 0, "max": 1, "mod-add": 2}
ROUTE = {"bdbs": 0, "bdbsc": 1, "box-complement": 2, "sat": 3, "satc": 4, "corners": 5,
         "corners-spine": 6}
ABI_VERSION = 2

EXPORTS = (
    "exsum_abi_version",
    "exsum_last_error",
    "exsum_shard_bc_tail",
    "exsum_shard_idem_workspace_bytes",
    "exsum_shard_idem_marginals",
    "exsum_shard_idem_write",
    "exsum_workspace_bytes",
    "exsum_route_workspace_bytes",
    "exsum_route",
    "exsum_route_host",
    "exsum_route_host_batch",
    "exsum_bdbs_included",
    "exsum_bdbsc_excluded",
    "exsum_box_complement_excluded",
    "exsum_windowed_pass",
    "exsum_run_host",
    "exsum_release_cache",
    "exsum_last_launch_count",
    "exsum_total_launch_count",
    "exsum_profile_enable",
    "exsum_profile_count",
    "exsum_profile_get",
    "exsum_scan_workspace_bytes",
    "exsum_scan_axis",
    "exsum_add_contribution",
    "exsum_elementwise",
    "exsum_fold_workspace_bytes",
    "exsum_fold",
    "exsum_shard_workspace_bytes",
    "exsum_shard_axis0_pass",
    "exsum_bdbs_finish",
    "exsum_box_complement_finish",
)

_lock = threading.Lock()
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"native library {LIB_PATH} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        vp, ci, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        L.exsum_abi_version.restype = ci
        L.exsum_last_error.restype = ctypes.c_char_p
        L.exsum_last_launch_count.restype = ci
        L.exsum_total_launch_count.restype = ctypes.c_longlong
        L.exsum_workspace_bytes.argtypes = [ci, ci, ci, ci, i64p, i64p, ctypes.POINTER(sz)]
        L.exsum_workspace_bytes.restype = ci
        for name in ("exsum_bdbs_included", "exsum_bdbsc_excluded", "exsum_box_complement_excluded"):
            fn = getattr(L, name)
            fn.argtypes = [vp, vp, ci, ci, ci, i64p, i64p, vp, sz, vp]
            fn.restype = ci
        L.exsum_windowed_pass.argtypes = [vp, vp, ci, ci, ci, i64p, ci, ctypes.c_int64, vp]
        L.exsum_windowed_pass.restype = ci
        L.exsum_run_host.argtypes = [ci, vp, vp, ci, ci, ci, i64p, i64p]
        L.exsum_run_host.restype = ci
        i64 = ctypes.c_int64
        L.exsum_route_workspace_bytes.argtypes = [ci, ci, ci, i64, ci, i64p, i64p,
                                                  ctypes.POINTER(sz)]
        L.exsum_route_workspace_bytes.restype = ci
        L.exsum_route.argtypes = [ci, vp, vp, ci, ci, i64, ci, i64p, i64p, vp, sz, vp]
        L.exsum_route.restype = ci
        L.exsum_route_host.argtypes = [ci, vp, vp, ci, ci, i64, ci, i64p, i64p]
        L.exsum_route_host.restype = ci
        L.exsum_route_host_batch.argtypes = [ci, ci, ctypes.POINTER(vp), ctypes.POINTER(vp), ci,
                                             ci, i64, ci, i64p, i64p]
        L.exsum_route_host_batch.restype = ci
        L.exsum_scan_workspace_bytes.argtypes = [ci, ci, i64, ci, i64p, ci, ctypes.POINTER(sz)]
        L.exsum_scan_workspace_bytes.restype = ci
        L.exsum_scan_axis.argtypes = [vp, vp, ci, ci, i64, ci, i64p, ci, ci, vp, sz, vp]
        L.exsum_scan_axis.restype = ci
        L.exsum_add_contribution.argtypes = [vp, vp, ci, ci, i64, ci, i64p, ci, i64, vp]
        L.exsum_add_contribution.restype = ci
        L.exsum_elementwise.argtypes = [vp, vp, vp, ci, ci, i64, ci, i64, vp]
        L.exsum_elementwise.restype = ci
        L.exsum_fold_workspace_bytes.restype = sz
        L.exsum_fold.argtypes = [vp, vp, ci, ci, i64, i64, vp, sz, vp]
        L.exsum_fold.restype = ci
        L.exsum_release_cache.restype = ci
        L.exsum_profile_enable.argtypes = [ci]
        L.exsum_profile_enable.restype = ci
        L.exsum_profile_count.restype = ci
        L.exsum_profile_get.argtypes = [ci, ctypes.c_char_p, ci, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_float)]
        L.exsum_profile_get.restype = ci
        L.exsum_shard_workspace_bytes.argtypes = [ci, ci, ci, ci, i64p, i64p, ctypes.c_int64, ci,
                                                  ctypes.POINTER(sz)]
        L.exsum_shard_workspace_bytes.restype = ci
        L.exsum_shard_axis0_pass.argtypes = [vp, vp, ci, ci, ci, i64p, i64p, ctypes.c_int64, ci, vp,
                                             vp, sz, vp]
        L.exsum_shard_axis0_pass.restype = ci
        for name in ("exsum_bdbs_finish", "exsum_box_complement_finish"):
            fn = getattr(L, name)
            fn.argtypes = [vp, vp, ci, ci, ci, i64p, i64p, vp, vp, sz, vp]
            fn.restype = ci
        L.exsum_shard_bc_tail.argtypes = [ci, vp, vp, vp, ci, ci, i64, i64, i64, i64, i64, i64, vp]
        L.exsum_shard_bc_tail.restype = ci
        L.exsum_shard_idem_workspace_bytes.argtypes = [ci, ci, ci, i64p, ctypes.POINTER(sz)]
        L.exsum_shard_idem_workspace_bytes.restype = ci
        L.exsum_shard_idem_marginals.argtypes = [vp, vp, ci, ci, ci, i64p, i64, i64, vp, sz, vp]
        L.exsum_shard_idem_marginals.restype = ci
        L.exsum_shard_idem_write.argtypes = [vp, vp, ci, ci, ci, i64p, i64p, i64, i64, vp]
        L.exsum_shard_idem_write.restype = ci
        if L.exsum_abi_version() != ABI_VERSION:
            raise DeviceError("libexsum_b200.so ABI version mismatch")
        _lib = L
        return L


def i64_array(seq):
    return (ctypes.c_int64 * len(seq))(*[int(v) for v in seq])


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load().exsum_last_error() or b"").decode(errors="replace")
    if rc == 1:
        raise UsageError(msg)
    if rc == 2:
        raise ConfigurationError(msg)
    raise DeviceError(msg or f"native call failed with code {rc}")


def workspace_bytes(route: str, dtype: str, op: str, ext, box, modulus: int = 0) -> int:
    out = ctypes.c_size_t(0)
    check(load().exsum_route_workspace_bytes(ROUTE[route], DTYPE[dtype], OP[op], int(modulus),
                                             len(ext), i64_array(ext), i64_array(box),
                                             ctypes.byref(out)))
    return int(out.value)


def profile_enable(on: bool) -> None:
    load().exsum_profile_enable(1 if on else 0)


def profile_records():
    """[(kernel name, algorithmic bytes, ms)] recorded since profile_enable(True).

    Call after synchronizing the stream the work ran on."""
    L = load()
    out = []
    buf = ctypes.create_string_buffer(64)
    for i in range(L.exsum_profile_count()):
        b = ctypes.c_double(0)
        ms = ctypes.c_float(0)
        check(L.exsum_profile_get(i, buf, 64, ctypes.byref(b), ctypes.byref(ms)))
        out.append((buf.value.decode(), float(b.value), float(ms.value)))
    return out


def total_launch_count() -> int:
    return int(load().exsum_total_launch_count())


def last_launch_count() -> int:
    return int(load().exsum_last_launch_count())
