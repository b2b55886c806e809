"""GPU parity for the outer pass pair (csrc/outer_pair.cu): the windowed
passes along two consecutive strided axes of extent 16 or 28 (scan.py:61-102,
in the order of included.py:124-129) in one kernel over strips of 128 bytes.
Same association as the single passes, so bdbs stays bit-identical to the
oracle and to EXSUM_OUTER_PAIR=0; bdbsc's complement rides on the pair's
stores when it is the last step.
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


def _run(ex, route, mono, arr, box, pair):
    import torch

    fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
          "box-complement": ex.box_complement_excluded}[route]
    old = os.environ.get("EXSUM_OUTER_PAIR")
    os.environ["EXSUM_OUTER_PAIR"] = str(pair)
    try:
        ops = ex.Float32AddOps() if mono == "add-f32" else ex.resolve_monoid(mono)
        data = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        out = fn(ex.Tensor(ops, data), box).data.cpu().numpy()
        n = ex._native.last_launch_count()
    finally:
        if old is None:
            del os.environ["EXSUM_OUTER_PAIR"]
        else:
            os.environ["EXSUM_OUTER_PAIR"] = old
    return out, n


def _data(rng, mono, shape):
    if mono == "add-f32":
        return rng.standard_normal(shape).astype(np.float32)
    if mono == "add-f64":
        return rng.standard_normal(shape)
    return rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)


def _bits(a, b):
    return a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


CASES = [
    ((28, 28, 64), (4, 4, 4)),
    ((28, 28, 32), (4, 4, 1)),          # the pair is the whole route
    ((3, 28, 28, 48), (1, 2, 2, 2)),
    ((16, 16, 32), (4, 4, 4)),
    ((2, 16, 16, 16, 16), (4, 4, 4, 4, 4)),
    ((28, 28, 28, 32), (4, 4, 4, 4)),
    ((16, 16, 64), (2, 2, 2)),
    ((28, 28, 32), (8, 8, 8)),           # float32 only (8-byte k = 8 takes the single passes)
    ((28, 28, 20), (4, 4, 4)),           # inner not a multiple of the 16-column strip: single passes
]


@pytest.mark.parametrize("shape,box", CASES, ids=lambda v: "x".join(map(str, v)))
@pytest.mark.parametrize("mono", ["add-f32", "add-i64", "max-i64", "add-f64"])
def test_outer_pair_bdbs(ex, shape, box, mono):
    rng = np.random.default_rng(sum(shape) + sum(box) + len(mono))
    a = _data(rng, mono, shape)
    op = "max" if mono == "max-i64" else "add"
    want = orc.ROUTES["bdbs"](a, box, op)
    got, n_pair = _run(ex, "bdbs", mono, a, box, 1)
    ref, n_single = _run(ex, "bdbs", mono, a, box, 0)
    assert _bits(got, want), (shape, box, mono)
    assert _bits(ref, want), (shape, box, mono)
    assert n_pair <= n_single


@pytest.mark.parametrize("shape,box", CASES[:4], ids=lambda v: "x".join(map(str, v)))
@pytest.mark.parametrize("mono", ["add-f32", "add-i64", "add-f64"])
def test_outer_pair_bdbsc_and_box_complement(ex, shape, box, mono):
    rng = np.random.default_rng(5 * sum(shape) + len(mono))
    a = _data(rng, mono, shape)
    for route in ("bdbsc", "box-complement"):
        got, _ = _run(ex, route, mono, a, box, 1)
        if a.dtype.kind == "i":
            assert _bits(got, orc.ROUTES[route](a, box, "add")), (route, shape, box, mono)
        else:
            ok, ratio, _ = compare(route, got, float64_oracle(route, a, box, orc), a, box, orc)
            assert ok, (route, shape, box, mono, ratio)


def test_outer_pair_taken_for_c3(ex):
    """28^5 / 16^6 float32 bdbs: one launch fewer with the pair, same bits."""
    rng = np.random.default_rng(1)
    for shape in [(28,) * 5, (16,) * 6]:
        a = rng.standard_normal(shape).astype(np.float32)
        box = (4,) * len(shape)
        got, n_pair = _run(ex, "bdbs", "add-f32", a, box, 1)
        ref, n_single = _run(ex, "bdbs", "add-f32", a, box, 0)
        assert _bits(got, ref), shape
        assert n_pair == n_single - 1, (shape, n_pair, n_single)
