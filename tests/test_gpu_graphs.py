"""CUDA-graph replay of repeated device calls (exsum_capi.cu run_device_graph):
a call repeated with the same route, shape, box and buffers is captured on
its second sighting and replayed after.  Replays must read the buffers'
CURRENT contents (new data in the same tensor -> the new result), report the
same launch count, and a changed EXSUM_* knob must not replay a stale plan.
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


@pytest.mark.parametrize("route,mono", [("box-complement", "max-i64"), ("bdbsc", "add-i64"),
                                        ("bdbs", "add-i64")])
def test_replay_reads_current_data(ex, route, mono):
    import torch

    from paper_2106_00124_b200.routes import run_device

    shape, box = (40, 24, 256), (8, 8, 8)
    x = torch.empty(shape, dtype=torch.int64, device="cuda")
    out = torch.empty_like(x)
    op = "max" if mono.startswith("max") else "add"
    counts = []
    for i in range(6):
        a = np.random.default_rng(i).integers(-2**30, 2**30, size=shape, dtype=np.int64)
        x.copy_(torch.from_numpy(a))
        run_device(route, x, "int64", op, shape, box, out=out)
        counts.append(ex._native.last_launch_count())
        assert np.array_equal(out.cpu().numpy(), orc.ROUTES[route](a, box, op)), (route, i)
    assert len(set(counts)) == 1 and counts[0] >= 1, counts


def test_env_knob_is_part_of_the_key(ex):
    import torch

    from paper_2106_00124_b200.routes import run_device

    shape, box = (6, 28, 28, 28), (4, 4, 4, 4)
    a = np.random.default_rng(3).standard_normal(shape).astype(np.float32)
    x = torch.from_numpy(a).cuda()
    out = torch.empty_like(x)
    want = orc.bdbs_included(a, box)
    n = {}
    for setting in ("1", "0", "1", "0", "1", "0"):
        os.environ["EXSUM_BLOCK_FUSE"] = setting
        try:
            run_device("bdbs", x, "float32", "add", shape, box, out=out)
        finally:
            del os.environ["EXSUM_BLOCK_FUSE"]
        n.setdefault(setting, set()).add(ex._native.last_launch_count())
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
    assert len(n["1"]) == 1 and len(n["0"]) == 1 and n["1"] != n["0"], n
