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


def _complement_fold(x, pt, box, op):
    """The fold of x over every cell outside the box at pt, as disjoint slab
    views (no copies): axis by axis, the cells before and after the box along
    that axis within the box's span on the earlier axes."""
    import torch

    parts = []
    pre = ()
    for a, (p, k) in enumerate(zip(pt, box)):
        n = x.shape[a]
        lo, hi = p, min(p + k, n)
        for sl in (slice(0, lo), slice(hi, n)):
            v = x[pre + (sl,)]
            if v.numel():
                parts.append(v.amax() if op == "max" else v.double().sum())
        pre = pre + (slice(lo, hi),)
    if not parts:
        return None
    t = torch.stack(parts)
    return t.amax() if op == "max" else t.sum()


def test_idem_max_past_2p31(ex):
    """Box-complement max through the marginal form (idem_max.cu) on 2.5e9
    int64 elements (sum of extents 4096, the form's limit): sampled points
    against the fold of their complement slabs, exactly."""
    import torch

    from paper_2106_00124_b200 import _native

    if _free_gb() < 50:
        pytest.skip("needs ~50 GB of free HBM")
    shape, box = (1366, 1366, 1364), (8, 8, 8)  # 2.55e9 elements, 20 GB
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randint(-2**40, 2**40, shape, generator=g, device="cuda", dtype=torch.int64)
    _native.profile_enable(True)
    out = ex.box_complement_excluded(ex.Tensor(ex.IntMaxOps(), x), box).data
    torch.cuda.synchronize()
    names = {n for n, _, _ in _native.profile_records()}
    _native.profile_enable(False)
    assert "idem_bcast" in names, names
    rng = np.random.default_rng(8)
    pts = [tuple(int(rng.integers(0, n)) for n in shape) for _ in range(24)]
    pts += [(0, 0, 0), (1365, 1365, 1363), (1359, 0, 1356), (683, 1362, 5)]
    for pt in pts:
        want = _complement_fold(x, pt, box, "max")
        assert int(out[pt]) == int(want), pt
    del out, x
    torch.cuda.empty_cache()


def test_box_complement_f32_past_2p31(ex):
    """The C4 route (axis pass with row partials, 3-D tail, strong row round)
    on 2.16e9 float32 elements: sampled points against the float64 fold of
    their complement, within the box-complement contract of tests/parity.py
    (values are >= 0, so S = BC(|A|) is the exact result itself)."""
    import torch

    if _free_gb() < 30:
        pytest.skip("needs ~30 GB of free HBM")
    shape, box = (2064, 1024, 1024), (16, 16, 16)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.rand(shape, generator=g, device="cuda")
    out = ex.box_complement_excluded(ex.Tensor(ex.Float32AddOps(), x), box).data
    torch.cuda.synchronize()
    from parity import U, depth, depth_ref

    tau = (depth("box-complement", shape, box) * U[np.dtype(np.float32)]
           + depth_ref("box-complement", shape, box) * 2.0**-53)
    rng = np.random.default_rng(10)
    pts = [tuple(int(rng.integers(0, n)) for n in shape) for _ in range(16)]
    pts += [(0, 0, 0), (2063, 1023, 1023), (2050, 7, 1015)]
    for pt in pts:
        want = float(_complement_fold(x, pt, box, "add"))
        tol = tau * want
        assert abs(float(out[pt]) - want) <= tol, (pt, float(out[pt]), want, tol)
    del out, x
    torch.cuda.empty_cache()
