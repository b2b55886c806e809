"""The tiled pass pair (csrc/tile_pair.cu): the last two BDBS passes with
window 32 in one launch (C1: float64 1024^2, box 32^2; C5's 32^3 box).

Against the C oracle (the reference's association, scan.py:61-102 along axes
0..d-1, included.py:124-129): BDBS bit-exact for every dtype, BDBSC bit-exact
for int64 and within the BDBSC contract of tests/parity.py for floats.
Edge shapes: extents not multiples of 32 or of the 128-column tile, the
k == n clamp, one- and many-tile arrays, an outer batch, a head pass before
the pair.  Every case also checks that the tiled kernel is the one that ran.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from parity import compare

pytestmark = pytest.mark.gpu

SHAPES = [
    ((1024, 1024), (32, 32)),   # C1
    ((32, 32), (32, 32)),       # one block each way: W = whole-axis suffix
    ((33, 40), (32, 32)),       # one-element / 8-element tail blocks
    ((64, 130), (32, 32)),      # a 2-column tail tile
    ((100, 260), (32, 32)),
    ((97, 300), (32, 32)),
    ((45, 34), (32, 32)),
    ((45, 33), (32, 32)),       # rows not a multiple of 16 bytes (element-granular staging)
    ((3, 70, 200), (1, 32, 32)),   # outer batch, no axis-0 pass
    ((5, 40, 96), (4, 32, 32)),    # head pass along axis 0, then the pair
    ((2, 3, 64, 160), (2, 1, 32, 32)),
]

MONOIDS = [("add-f64", np.float64), ("add-f32", np.float32), ("add-i64", np.int64),
           ("max-i64", np.int64)]


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _ops(ex, name):
    return {"add-f64": ex.FloatAddOps, "add-f32": ex.Float32AddOps, "add-i64": ex.IntAddOps,
            "max-i64": ex.IntMaxOps}[name]()


def _input(shape, dt, seed):
    rng = np.random.default_rng(seed)
    if dt == np.int64:
        return rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)
    return rng.standard_normal(shape).astype(dt)


def _tiled(a):
    """Every case here takes the tiled kernel (window 32, <= 64 MB)."""
    return True


def _run(ex, fn, mono, a):
    import torch

    from paper_2106_00124_b200 import _native

    t = ex.Tensor(mono, torch.from_numpy(a).cuda())
    _native.profile_enable(True)
    got = fn(t).data
    torch.cuda.synchronize()
    names = [n for n, _, _ in _native.profile_records()]
    _native.profile_enable(False)
    return got.cpu().numpy(), names


@pytest.mark.parametrize("shape,box", SHAPES)
@pytest.mark.parametrize("mname,dt", MONOIDS)
def test_tile_pair_bdbs(ex, shape, box, mname, dt):
    a = _input(shape, dt, 7)
    op = "max" if mname == "max-i64" else "add"
    got, names = _run(ex, lambda t: ex.bdbs_included(t, box), _ops(ex, mname), a)
    assert ("tile_pair" in names) == _tiled(a), names
    want = orc.bdbs_included(a, box, op)
    assert got.dtype == want.dtype
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("shape,box", SHAPES)
@pytest.mark.parametrize("mname,dt", [m for m in MONOIDS if m[0] != "max-i64"])
def test_tile_pair_bdbsc(ex, shape, box, mname, dt):
    a = _input(shape, dt, 11)
    got, names = _run(ex, lambda t: ex.bdbs_excluded(t, box), _ops(ex, mname), a)
    assert ("tile_pair" in names) == _tiled(a), names
    if dt == np.int64:
        assert np.array_equal(got, orc.bdbs_excluded(a, box, "add"))
    else:
        want = orc.bdbs_excluded(a.astype(np.float64), box, "add")
        ok, worst, _ = compare("bdbsc", got, want, a, box, orc)
        assert ok, worst
