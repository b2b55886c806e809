"""Box-complement for max as per-axis marginals (csrc/idem_max.cu).

For an idempotent operator the complement of a box is the union of the 2d
half-space slabs, so the strong excluded sum factorises into per-axis 1-D
excluded windows of the marginals (see the kernel file).  It must be
bit-identical to the reference's slab algorithm (excluded.py:129-159) as
restated by the C oracle, on every shape and box the route accepts: k = 1,
k >= n (clamped: empty complement along that axis, identity everywhere when
every axis is clamped), one-element axes, odd rows (the scalar path), views
off 16-byte alignment, values at the int64 extremes, d = 2..5.
"""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

I64_MIN = np.iinfo(np.int64).min
I64_MAX = np.iinfo(np.int64).max

CASES = [
    ((256, 256, 256), (8, 8, 8)),      # C2
    ((64, 48, 40), (8, 8, 8)),
    ((17, 33, 65), (4, 5, 7)),         # odd rows: scalar path
    ((16, 16, 16), (16, 16, 16)),      # every axis clamped: empty complement
    ((16, 16, 16), (16, 1, 16)),
    ((20, 30), (1, 1)),                # k = 1: the complement is all but x
    ((1, 50, 64), (3, 8, 8)),          # one-element axis
    ((300, 2), (7, 5)),                # k > n on the last axis
    ((9, 7, 6, 10), (2, 3, 4, 5)),
    ((4, 5, 6, 7, 8), (2, 2, 3, 3, 4)),
    ((1000, 1000), (32, 32)),
    ((2, 3000), (1, 100)),
    ((50, 40, 1), (3, 4, 1)),          # a one-element last axis
    ((1, 1, 300), (1, 1, 9)),          # only the last axis varies
    ((7, 1, 5, 1, 9), (2, 1, 3, 1, 4)),
    ((4000, 3, 2), (17, 2, 1)),        # many short rows
]


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _run(ex, a, box, offset=0):
    import torch

    from paper_2106_00124_b200 import _native

    if offset:
        buf = torch.empty(a.size + offset, dtype=torch.int64, device="cuda")
        x = buf[offset:].view(a.shape)
        x.copy_(torch.from_numpy(a))
    else:
        x = torch.from_numpy(a).cuda()
    t = ex.Tensor(ex.IntMaxOps(), x)
    _native.profile_enable(True)
    got = ex.box_complement_excluded(t, box).data
    torch.cuda.synchronize()
    names = [n for n, _, _ in _native.profile_records()]
    _native.profile_enable(False)
    return got.cpu().numpy(), names


@pytest.mark.parametrize("shape,box", CASES)
def test_idem_max_matches_slab_oracle(ex, shape, box):
    rng = np.random.default_rng(3)
    a = rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)
    got, names = _run(ex, a, box)
    assert "idem_scan" in names and "idem_bcast" in names, names
    assert np.array_equal(got, orc.box_complement_excluded(a, box, "max"))


@pytest.mark.parametrize("offset", [1, 3])
def test_idem_max_unaligned_view(ex, offset):
    rng = np.random.default_rng(offset)
    a = rng.integers(-1000, 1000, size=(24, 40, 66), dtype=np.int64)
    got, _ = _run(ex, a, (4, 8, 8), offset=offset)
    assert np.array_equal(got, orc.box_complement_excluded(a, (4, 8, 8), "max"))


def test_idem_max_extremes(ex):
    rng = np.random.default_rng(9)
    a = rng.choice(np.array([I64_MIN, I64_MIN + 1, -1, 0, 1, I64_MAX - 1, I64_MAX], np.int64),
                   size=(33, 20, 18))
    a[0, 0, 0] = I64_MAX
    got, _ = _run(ex, a, (5, 4, 3))
    assert np.array_equal(got, orc.box_complement_excluded(a, (5, 4, 3), "max"))
    # a single maximum: every output whose box misses it equals it
    b = np.full((12, 12, 12), I64_MIN, np.int64)
    b[6, 6, 6] = 42
    got, _ = _run(ex, b, (3, 3, 3))
    assert np.array_equal(got, orc.box_complement_excluded(b, (3, 3, 3), "max"))


def test_idem_max_c2_full_size_seeded(ex):
    """C2 on bench.py's own seeded input, against the slab oracle."""
    import bench

    x = bench.make_input("c2", "cuda", seed=0)
    a = x.cpu().numpy()
    got, _ = _run(ex, a, (8, 8, 8))
    assert np.array_equal(got, orc.box_complement_excluded(a, (8, 8, 8), "max", 0))


def test_idem_max_large_tables_take_the_slab_route(ex):
    """Extents summing past the marginal tables' bound run the slab route."""
    rng = np.random.default_rng(5)
    a = rng.integers(-2**40, 2**40, size=(4200, 3), dtype=np.int64)
    got, names = _run(ex, a, (7, 2))
    assert "idem_scan" not in names, names
    assert np.array_equal(got, orc.box_complement_excluded(a, (7, 2), "max"))
