"""GPU parity for the trailing-block fusion (csrc/block_fused.cu): the
windowed passes of the last m axes of bdbs_included (included.py:124-129,
scan.py:61-102) run in shared memory in one kernel when a block of those axes
fits.  The fused kernel keeps the reference's association, so float bdbs stays
bit-identical to the oracle and to the unfused passes (EXSUM_BLOCK_FUSE=0);
bdbsc carries the complement epilogue on the fused kernel's stores.

Every dtype takes the fused kernel where the plan allows (EXSUM_BLOCK_FUSE=1,
the default; 2 is the same plan, kept as the explicit "all dtypes" switch).
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc
from parity import compare, float64_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _mono(ex, name):
    return ex.Float32AddOps() if name == "add-f32" else ex.resolve_monoid(name)


def _run(ex, route, mono, arr, box, fuse):
    import torch

    fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded}[route]
    old = os.environ.get("EXSUM_BLOCK_FUSE")
    os.environ["EXSUM_BLOCK_FUSE"] = str(fuse)
    try:
        data = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        out = fn(ex.Tensor(_mono(ex, mono), data), box).data.cpu().numpy()
        launches = ex._native.last_launch_count()
    finally:
        if old is None:
            del os.environ["EXSUM_BLOCK_FUSE"]
        else:
            os.environ["EXSUM_BLOCK_FUSE"] = old
    return out, launches


def _bits_equal(a, b):
    return a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def _data(rng, mono, shape):
    if mono == "add-f32":
        return rng.standard_normal(shape).astype(np.float32)
    if mono == "add-f64":
        return rng.standard_normal(shape)
    return rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)


CASES = [
    # (shape, box): the C3 shapes scaled down, tails (n % k != 0), k = 1 axes,
    # k >= n (clamped), extents of 1, several blocks per CTA tile, odd rows
    ((6, 28, 28, 28), (4, 4, 4, 4)),
    ((3, 16, 16, 16, 16), (4, 4, 4, 4, 4)),
    ((5, 64, 64), (4, 4, 4)),
    ((7, 13, 11), (4, 1, 4)),
    ((9, 10, 17), (2, 2, 2)),
    ((4, 3, 5, 7), (4, 4, 4, 4)),
    ((2, 9, 1, 6), (8, 8, 1, 8)),
    ((33, 30, 30), (8, 8, 8)),
    ((1, 12, 12), (4, 4, 4)),
    ((100, 5), (4, 4)),
]


@pytest.mark.parametrize("shape,box", CASES)
@pytest.mark.parametrize("mono", ["add-f32", "add-i64", "max-i64", "add-f64"])
def test_block_fused_bdbs_exact(ex, shape, box, mono):
    rng = np.random.default_rng(sum(shape) + len(mono))
    a = _data(rng, mono, shape)
    op = "max" if mono == "max-i64" else "add"
    got, n_fused = _run(ex, "bdbs", mono, a, box, fuse=2)
    ref, n_plain = _run(ex, "bdbs", mono, a, box, fuse=0)
    want = orc.ROUTES["bdbs"](a, box, op)
    assert _bits_equal(got, want), (shape, box, mono)
    assert _bits_equal(ref, want), (shape, box, mono)
    assert n_fused <= n_plain


@pytest.mark.parametrize("shape,box", CASES[:6])
@pytest.mark.parametrize("mono", ["add-f32", "add-i64", "add-f64"])
def test_block_fused_bdbsc(ex, shape, box, mono):
    rng = np.random.default_rng(7 * sum(shape) + len(mono))
    a = _data(rng, mono, shape)
    got, _ = _run(ex, "bdbsc", mono, a, box, fuse=2)
    if a.dtype.kind == "i":
        assert _bits_equal(got, orc.ROUTES["bdbsc"](a, box, "add")), (shape, box, mono)
    else:
        k = tuple(min(b, e) for b, e in zip(box, shape))
        ok, ratio, rel = compare("bdbsc", got, float64_oracle("bdbsc", a, k, orc), a, k, orc)
        assert ok, (shape, box, mono, ratio)


@pytest.mark.parametrize("mono", ["add-f32", "max-i64"])
def test_block_fused_is_taken_for_c3_shapes(ex, mono):
    """The C3 shapes of higher dimension (float32 +, int64 max) run the fused
    kernel by default (fewer launches than the unfused passes) with identical bits."""
    rng = np.random.default_rng(3)
    for shape in [(28,) * 5, (16,) * 6, (64,) * 4]:
        a = _data(rng, mono, shape)
        box = (4,) * len(shape)
        got, n_fused = _run(ex, "bdbs", mono, a, box, fuse=1)
        ref, n_plain = _run(ex, "bdbs", mono, a, box, fuse=0)
        assert _bits_equal(got, ref), shape
        assert n_fused < n_plain, (shape, n_fused, n_plain)


def _run_env(ex, route, mono, arr, box, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return _run(ex, route, mono, arr, box, fuse=1)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


# cubic trailing blocks take k_block_cubic<NL, M> (compile-time line length,
# strides and layout: odd vector stride, XOR-swizzled 64-byte rows, padded
# planes); every NL / M form, every window, skipped axes (k = 1) inside the
# block, tiles of several blocks, against the oracle and the runtime-shape
# kernel (EXSUM_BF_CUBIC=0)
# leading extents large enough that the plan stops at the cubic block (a
# small leading axis would join the block and take the runtime-shape kernel)
CUBIC = [
    ((7, 16, 16, 16), (2, 2, 2, 2)),
    ((7, 16, 16, 16), (4, 1, 4, 4)),
    ((2, 16, 16, 16, 16), (4, 4, 4, 1, 4)),
    ((4, 28, 28, 28), (4, 4, 4, 4)),
    ((4, 28, 28, 28), (2, 2, 1, 2)),
    ((200, 28, 28), (4, 4, 4)),
    ((120, 32, 32), (2, 2, 2)),
    ((120, 32, 32), (4, 4, 4)),
    ((9, 64, 64), (4, 4, 4)),
    ((9, 64, 64), (2, 2, 1)),
    ((3, 28, 28, 28), (8, 8, 8, 8)),
    ((7, 16, 16, 16), (8, 8, 8, 8)),
]


@pytest.mark.parametrize("shape,box", CUBIC, ids=lambda v: "x".join(map(str, v)))
@pytest.mark.parametrize("mono", ["add-f32", "add-i64", "max-i64", "add-f64"])
def test_block_cubic_forms(ex, shape, box, mono):
    rng = np.random.default_rng(11 * sum(shape) + sum(box) + len(mono))
    a = _data(rng, mono, shape)
    op = "max" if mono == "max-i64" else "add"
    want = orc.ROUTES["bdbs"](a, box, op)
    got, _ = _run_env(ex, "bdbs", mono, a, box, {"EXSUM_BF_CUBIC": "1"})
    gen, _ = _run_env(ex, "bdbs", mono, a, box, {"EXSUM_BF_CUBIC": "0"})
    assert _bits_equal(got, want), (shape, box, mono)
    assert _bits_equal(gen, want), (shape, box, mono)
    if mono != "max-i64":
        gotc, _ = _run_env(ex, "bdbsc", mono, a, box, {"EXSUM_BF_CUBIC": "1"})
        if a.dtype.kind == "i":
            assert _bits_equal(gotc, orc.ROUTES["bdbsc"](a, box, "add")), (shape, box, mono)
        else:
            ok, ratio, _ = compare("bdbsc", gotc, float64_oracle("bdbsc", a, box, orc), a, box, orc)
            assert ok, (shape, box, mono, ratio)
