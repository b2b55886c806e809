"""GPU parity for the opt-in L2-pipelined schedule (csrc/l2pipe.cu,
EXSUM_L2PIPE=1): one persistent kernel in which producer CTAs run the axis-0
pass into an L2-resident ring and consumer CTAs run the fused pass pair from
it.  Same kernels' association as the default two-kernel schedule, so bdbs is
bit-identical to it and to the oracle; box-complement differs only through
the order of the R fold (a pre-pass here), inside the float tolerance.
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


def _run(ex, fn, a, box, pipe):
    import torch

    old = os.environ.get("EXSUM_L2PIPE")
    os.environ["EXSUM_L2PIPE"] = "1" if pipe else "0"
    ex.routes._PLAN_CACHE.clear()  # the workspace size depends on the schedule
    try:
        x = torch.from_numpy(a).cuda()
        out = fn(ex.Tensor(ex.Float32AddOps(), x), box).data.cpu().numpy()
        n = ex._native.last_launch_count()
    finally:
        if old is None:
            del os.environ["EXSUM_L2PIPE"]
        else:
            os.environ["EXSUM_L2PIPE"] = old
        ex.routes._PLAN_CACHE.clear()
    return out, n


@pytest.mark.parametrize("shape", [(64, 96, 1024), (48, 64, 1024), (32, 208, 1024)])
def test_l2pipe_bdbs_bit_exact(ex, shape):
    a = np.random.default_rng(sum(shape)).standard_normal(shape).astype(np.float32)
    box = (16, 16, 16)
    got, n_pipe = _run(ex, ex.bdbs_included, a, box, True)
    ref, n_two = _run(ex, ex.bdbs_included, a, box, False)
    assert n_pipe == 1 and n_two == 2  # the pipelined kernel actually ran
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(got.view(np.uint32), orc.ROUTES["bdbs"](a, box, "add").view(np.uint32))


@pytest.mark.parametrize("shape", [(64, 96, 1024), (32, 208, 1024)])
def test_l2pipe_box_complement(ex, shape):
    a = np.random.default_rng(7 + sum(shape)).random(shape, dtype=np.float32)
    box = (16, 16, 16)
    got, _ = _run(ex, ex.box_complement_excluded, a, box, True)
    ok, ratio, rel = compare("box-complement", got, float64_oracle("box-complement", a, box, orc),
                             a, box, orc)
    assert ok, ratio
