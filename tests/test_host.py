"""Host-side logic and the C-ABI boundary (CPU only; no kernel is executed)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2106_00124_b200 as ex
from paper_2106_00124_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "exsum_b200.h")).read()
    return re.findall(r"^\s*(?:const\s+)?(?:long\s+)?\w+\s*\*?\s*(exsum_\w+)\s*\(", text, re.M)


def test_library_exports_every_header_symbol():
    L = _native.load()
    names = _header_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_native.EXPORTS)
    assert L.exsum_abi_version() == 2


def test_library_is_sm100a():
    blob = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_error_classes_mirror_reference():
    assert issubclass(ex.UsageError, ValueError)
    assert issubclass(ex.UsageError, ex.ExsumError)
    assert issubclass(ex.ConfigurationError, ex.ExsumError)
    assert issubclass(ex.VerificationError, ex.ExsumError)


def test_normalize_box_like_reference():
    assert ex.normalize_box((5, 5), (2, 9)) == (2, 5)
    with pytest.raises(ex.UsageError):
        ex.normalize_box((5, 5), (2,))
    with pytest.raises(ex.UsageError):
        ex.normalize_box((5, 5), (0, 1))
    with pytest.raises(ex.UsageError):
        ex.validate_extents((3, 0))
    with pytest.raises(ex.UsageError):
        ex.validate_extents(())


def test_validation_happens_before_any_device_work():
    t = ex.Tensor(ex.IntAddOps(), np.zeros((5, 5), dtype=np.int64))
    with pytest.raises(ex.UsageError):
        ex.bdbs_included(t, (2,))
    with pytest.raises(ex.UsageError):
        ex.box_complement_excluded(t, (2, 2, 2))
    with pytest.raises(ex.UsageError):
        ex.bdbs_excluded(t, (0, 1))
    tm = ex.Tensor(ex.IntMaxOps(), np.zeros((5, 5), dtype=np.int64))
    with pytest.raises(ex.ConfigurationError):
        ex.bdbs_excluded(tm, (2, 2))
    with pytest.raises(ex.ConfigurationError):
        ex.resolve_monoid("mod-add:1")
    for route in (ex.sat_included, ex.sat_excluded):
        with pytest.raises(ex.ConfigurationError):
            route(tm, (2, 2))
        with pytest.raises(ex.UsageError):
            route(t, (2, 2, 2))


def test_unsupported_monoid_is_configuration_error():
    class Weird:
        name = "xor-i64"
        dtype = np.dtype(np.int64)
        identity = 0

    t = ex.Tensor(Weird(), np.zeros((3,), dtype=np.int64))
    with pytest.raises(ex.ConfigurationError):
        ex.bdbs_included(t, (2,))

    class RefMod:  # duck-typed like the reference's ModAddOps: modulus from the name
        name = "mod-add:11"
        dtype = np.dtype(np.int64)
        identity = 0
        has_inverse = True

    from paper_2106_00124_b200.monoid import modulus_of

    assert modulus_of(RefMod()) == 11
    RefMod.name = "mod-add:1"
    with pytest.raises(ex.ConfigurationError):
        ex.bdbs_included(ex.Tensor(RefMod(), np.zeros((3,), dtype=np.int64)), (2,))


def test_reference_style_monoids_and_instrumentation_unwrap():
    class RefAdd:  # duck-typed like exsum.IntAddOps
        name = "add-i64"
        dtype = np.dtype(np.int64)
        identity = 0
        has_inverse = True

    class Instrumented:  # like exsum.InstrumentedMonoid (bench.py:128 unwraps .inner)
        def __init__(self, inner):
            self.inner = inner
            self.name = inner.name
            self.dtype = inner.dtype

    from paper_2106_00124_b200.monoid import device_operator

    assert device_operator(RefAdd()) == (np.dtype(np.int64), "add", True)
    assert device_operator(Instrumented(RefAdd())) == (np.dtype(np.int64), "add", True)
    assert device_operator(ex.IntMaxOps()) == (np.dtype(np.int64), "max", False)
    assert device_operator(ex.Float32AddOps())[0] == np.dtype(np.float32)
    assert device_operator(ex.ModAddOps(97)) == (np.dtype(np.int64), "mod-add", True)
    assert device_operator(ex.resolve_monoid("mod-add:13"))[1] == "mod-add"
    for bad in ("mod-add:1", "mod-add:x", "mod-add:", "sum"):
        with pytest.raises(ex.ConfigurationError):
            ex.resolve_monoid(bad)
    with pytest.raises(ex.ConfigurationError):
        ex.ModAddOps(2**31 + 1)
    assert ex.ModAddOps(2**31).combine(2**31 - 1, 1) == 0
    assert ex.ModAddOps(5).subtract(1, 3) == 3


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = ex.Tensor(ex.IntAddOps(), np.arange(12, dtype=np.int64).reshape(3, 4))
    with pytest.raises(ex.DeviceError):
        ex.bdbs_included(t, (2, 2))


def test_c_abi_validation_codes():
    L = _native.load()
    ext = _native.i64_array((4, 4))
    box = _native.i64_array((2, 2))
    out = ctypes.c_size_t(0)
    assert L.exsum_workspace_bytes(0, 0, 0, 2, ext, box, ctypes.byref(out)) == 0
    assert L.exsum_workspace_bytes(1, 2, 1, 2, ext, box, ctypes.byref(out)) == 2  # bdbsc + max
    assert L.exsum_workspace_bytes(0, 1, 1, 2, ext, box, ctypes.byref(out)) == 2  # max-f64
    assert L.exsum_workspace_bytes(0, 7, 0, 2, ext, box, ctypes.byref(out)) == 2  # dtype
    assert L.exsum_workspace_bytes(0, 0, 0, 0, ext, box, ctypes.byref(out)) == 1  # d = 0
    bad = _native.i64_array((0, 2))
    assert L.exsum_workspace_bytes(0, 0, 0, 2, ext, bad, ctypes.byref(out)) == 1  # k = 0
    assert b"box side" in L.exsum_last_error()
    # device entry points refuse aliasing and null pointers before touching CUDA
    assert L.exsum_bdbs_included(None, None, 0, 0, 2, ext, box, None, 0, None) == 1
    assert L.exsum_bdbs_included(16, 16, 0, 0, 2, ext, box, None, 0, None) == 1
    # sat / satc need an inverse; mod-add needs int64 and 2 <= m <= 2^31
    rw = L.exsum_route_workspace_bytes
    assert rw(3, 2, 1, 0, 2, ext, box, ctypes.byref(out)) == 2  # sat + max
    assert b"'sat' requires an invertible" in L.exsum_last_error()
    assert rw(4, 2, 1, 0, 2, ext, box, ctypes.byref(out)) == 2  # satc + max
    assert rw(7, 2, 0, 0, 2, ext, box, ctypes.byref(out)) == 2  # no route 7
    assert rw(5, 2, 1, 0, 2, ext, box, ctypes.byref(out)) == 0  # corners, max, 2-D
    one = _native.i64_array((4,))
    assert rw(5, 2, 0, 0, 1, one, one, ctypes.byref(out)) == 2  # corners, 1-D
    assert b"2-D and 3-D" in L.exsum_last_error(), L.exsum_last_error()
    assert rw(3, 2, 0, 0, 2, ext, box, ctypes.byref(out)) == 0  # sat add-i64
    for m, want in ((1, 2), (2, 0), (2**31, 0), (2**31 + 1, 2)):
        assert rw(2, 2, 2, m, 2, ext, box, ctypes.byref(out)) == want, m
    assert rw(0, 0, 2, 7, 2, ext, box, ctypes.byref(out)) == 2  # mod-add on float32
    assert L.exsum_workspace_bytes(0, 2, 2, 2, ext, box, ctypes.byref(out)) == 2  # no modulus
    assert L.exsum_route(0, None, None, 2, 2, 7, 2, ext, box, None, 0, None) == 1


def test_workspace_sizes():
    # BDBS with >= 2 active passes needs one ping-pong array
    n = 1 << 30
    assert _native.workspace_bytes("bdbs", "float32", "add", (1024,) * 3, (16,) * 3) == 4 * n
    assert _native.workspace_bytes("bdbs", "float32", "add", (1024, 1024), (1, 16)) == 0
    # box-complement: W buffer + per-level reductions (<= N + small)
    ws = _native.workspace_bytes("box-complement", "float32", "add", (1024,) * 3, (16,) * 3)
    assert 4 * n <= ws <= 4 * n + 256 * 2**20  # W buffer + row partials + per-level reductions
    # sat: the running-sum table; satc adds the reduction partials
    assert _native.workspace_bytes("sat", "float32", "add", (1024,) * 3, (16,) * 3) == 4 * n
    assert 4 * n < _native.workspace_bytes("satc", "float32", "add", (1024,) * 3, (16,) * 3) \
        <= 4 * n + 2**20
    # mod-add: canonical residues + the int64 route's own workspace
    m = _native.workspace_bytes("bdbs", "int64", "mod-add", (256,) * 3, (8,) * 3, 97)
    assert 2 * 8 * 256**3 <= m <= 2 * 8 * 256**3 + 2**20
    # a long 1-D axis is scanned in segments (carry buffer, a few KB)
    seg = _native.workspace_bytes("sat", "float64", "add", (1 << 22,), (5,))
    assert 8 << 22 < seg < (8 << 22) + 2**20


def test_registry_mirrors_reference():
    assert set(ex.ALGORITHMS) == {"sat", "bdbs", "satc", "bdbsc", "box-complement", "corners",
                                  "corners-spine"}
    assert ex.resolve_algorithm("corners").cache_arg == "buffers"
    assert ex.resolve_algorithm("corners-spine").cache_arg == "cache_depth"
    with pytest.raises(ex.ConfigurationError):
        ex.check_algorithm_config(ex.resolve_algorithm("corners"), ex.IntAddOps(), 4)
    t1 = ex.Tensor(ex.IntAddOps(), np.zeros(5, dtype=np.int64))
    t2 = ex.Tensor(ex.IntAddOps(), np.zeros((3, 4), dtype=np.int64))
    with pytest.raises(ex.ConfigurationError):
        ex.corners_excluded(t1, (2,))
    with pytest.raises(ex.UsageError):
        ex.corners_excluded(t2, (2, 2), buffers=3)
    with pytest.raises(ex.UsageError):
        ex.corners_spine_excluded(t2, (2, 2), cache_depth=0)
    with pytest.raises(ex.UsageError):
        ex.corners_excluded(t2, (2,))
    for name in ("sat", "satc"):
        with pytest.raises(ex.ConfigurationError):
            ex.check_algorithm_config(ex.resolve_algorithm(name), ex.IntMaxOps())
        ex.check_algorithm_config(ex.resolve_algorithm(name), ex.ModAddOps(7))
    info = ex.resolve_algorithm("bdbsc")
    assert info.needs_inverse and info.kind == "excluded"
    with pytest.raises(ex.ConfigurationError):
        ex.check_algorithm_config(info, ex.IntMaxOps())
    ex.check_algorithm_config(ex.resolve_algorithm("box-complement"), ex.IntMaxOps())
    with pytest.raises(ex.ConfigurationError):
        ex.resolve_algorithm("naive-inc")  # not on the accelerated path


def test_register_with_reference_registry():
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class AlgorithmInfo:
        name: str
        fn: object
        kind: str
        needs_inverse: bool
        dims: object = None
        cache_arg: str = ""

    class FakeBench:
        pass

    fb = FakeBench()
    fb.AlgorithmInfo = AlgorithmInfo
    fb.ALGORITHMS = {"bdbs": None, "naive-inc": "untouched"}
    ex.register_with_reference(fb)
    assert fb.ALGORITHMS["bdbs"].fn is ex.bdbs_included
    assert fb.ALGORITHMS["box-complement"].fn is ex.box_complement_excluded
    assert fb.ALGORITHMS["sat"].fn is ex.sat_included and fb.ALGORITHMS["sat"].needs_inverse
    assert fb.ALGORITHMS["satc"].fn is ex.sat_excluded
    assert fb.ALGORITHMS["naive-inc"] == "untouched"
    assert fb.ALGORITHMS["corners"].cache_arg == "buffers" and fb.ALGORITHMS["corners"].dims == {2, 3}


def test_pad_and_crop():
    t = ex.Tensor(ex.IntAddOps(), np.arange(10, dtype=np.int64).reshape(2, 5))
    p, ext = ex.pad_to_box_multiple(t, (2, 3))
    assert p.extents == (2, 6) and ext == (2, 5)
    assert p.data[0, 5] == 0
    assert np.array_equal(ex.crop_to(p, ext).data, t.data)


def test_tensor_dtype_check():
    with pytest.raises(ex.UsageError):
        ex.Tensor(ex.IntAddOps(), np.zeros(3, dtype=np.float64))
