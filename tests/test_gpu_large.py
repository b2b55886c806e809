"""Maximum sizes: arrays past 2^31 elements (64-bit indexing in every kernel).

Full-size parity through size-independent properties (the oracle cannot run
17 GB in seconds): windowed sums are local along axis 0, so output planes
[a, b) equal the oracle on input planes [a, b + k0 - 1) (bit-exact, floats too,
when a is a multiple of k0); for int64 + the strong and weak excluded sums
agree exactly (box-complement == bdbsc) and sat == bdbs.
"""

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


def _free_gb():
    import torch

    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


def _slab_check(ex, x, out, box, op, planes):
    k0 = box[0]
    n0 = x.shape[0]
    for a in planes:
        b = min(a + 16, n0)
        src = x[a:min(b + k0 - 1, n0)].cpu().numpy()
        want = orc.bdbs_included(src, box, op)[: b - a]
        got = out[a:b].cpu().numpy()
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (a, b)


def test_bdbs_f32_past_2p31(ex):
    import torch

    if _free_gb() < 30:
        pytest.skip("needs ~30 GB of free HBM")
    shape, box = (2064, 1024, 1024), (16, 16, 16)  # 2.16e9 elements, 8.7 GB
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(shape, generator=g, device="cuda")
    out = ex.bdbs_included(ex.Tensor(ex.Float32AddOps(), x), box).data
    torch.cuda.synchronize()
    _slab_check(ex, x, out, box, "add", [0, 1024, 2048])
    del out, x
    torch.cuda.empty_cache()


def test_int64_routes_past_2p31(ex):
    import torch

    if _free_gb() < 90:
        pytest.skip("needs ~90 GB of free HBM")
    shape, box = (2056, 1024, 1024), (8, 8, 8)  # 2.16e9 elements, 17 GB
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randint(-2**20, 2**20, shape, generator=g, device="cuda", dtype=torch.int64)
    t = ex.Tensor(ex.IntAddOps(), x)
    inc = ex.bdbs_included(t, box).data
    torch.cuda.synchronize()
    _slab_check(ex, x, inc, box, "add", [0, 1040, 2040])
    sat = ex.sat_included(t, box).data
    assert torch.equal(sat, inc)
    del sat
    weak = ex.bdbs_excluded(t, box).data
    strong = ex.box_complement_excluded(t, box).data
    assert torch.equal(weak, strong)
    del weak, strong, inc
    tm = ex.Tensor(ex.IntMaxOps(), x)
    incm = ex.bdbs_included(tm, box).data
    torch.cuda.synchronize()
    _slab_check(ex, x, incm, box, "max", [0, 2048])
    del incm, x
    torch.cuda.empty_cache()
