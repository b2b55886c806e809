"""GPU parity of the BDBSC total when it rides on the first pass.

bdbs_excluded (excluded.py:72-75) needs the total of the input; the library
folds it into the first windowed pass (per-CTA partials + launch_total_final)
instead of a separate read.  Here the first pass is the TMA bulk kernel
(k > 16 for 8-byte, k > 32 for 4-byte elements, csrc/pass_bulk.cu): int64
bit-exact against the oracle, floats within the tests/parity.py bound, and one
launch fewer than with the total forced separate (EXSUM_STRIDED=reg takes the
register kernel, which carries partials as well, so the comparison is against
the oracle only).
"""

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


CASES = [
    ((300, 40, 64), (128, 4, 1), "add-f64"),
    ((300, 40, 64), (32, 32, 32), "add-f64"),
    ((200, 3, 96), (33, 2, 5), "add-i64"),
    ((150, 64), (100, 3), "add-f32"),
    ((512, 32), (128, 1), "add-i64"),
]


@pytest.mark.parametrize("shape,box,mono", CASES, ids=lambda v: str(v))
def test_bdbsc_total_on_bulk_pass(ex, shape, box, mono):
    import torch

    rng = np.random.default_rng(sum(shape) + sum(box))
    if mono == "add-i64":
        a = rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)
    else:
        a = rng.standard_normal(shape).astype(np.float32 if mono == "add-f32" else np.float64)
    ops = ex.Float32AddOps() if mono == "add-f32" else ex.resolve_monoid(mono)
    t = ex.Tensor(ops, torch.from_numpy(a).cuda())
    got = ex.bdbs_excluded(t, box).data.cpu().numpy()
    k = tuple(min(b, n) for b, n in zip(box, shape))
    if a.dtype.kind == "i":
        assert np.array_equal(got, orc.bdbs_excluded(a, k, "add"))
    else:
        ok, ratio, _ = compare("bdbsc", got, float64_oracle("bdbsc", a, k, orc), a, k, orc)
        assert ok, ratio
