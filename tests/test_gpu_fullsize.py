"""Full-size oracle parity on the BASELINE configs that the bench measures.

* C4 (float32 1024^3 uniform [0,1), box 16^3; bench.py's own seeded input):
  - box-complement against the float64 oracle on every plane of three
    plane bands (head, middle, tail).  The oracle side follows the
    reference's own decomposition (excluded.py:129-159, SURVEY App. A.3,
    peeling axis 0): for a plane x0,
        out[x0] = Win_{1,2}( P[x0-1] + S[x0+k0] ) + BC_2(R_1)
    with P / S the full-axis inclusive prefix / suffix of A along axis 0
    (sequential float64 folds over the planes, numpy's accumulate order),
    Win_{1,2} the windowed passes along axes 1, 2 (the windowed pass is
    linear, so the passes of the scanned planes equal the scans of the
    passed planes) and BC_2(R_1) the 2-D box complement of the column sums.
    The 2-D pieces are the C oracle's bdbs_included / box_complement_excluded.
    Tolerance: tests/parity.py's box-complement contract, S = BC(|A|) = the
    float64 answer itself (A >= 0).
  - BDBS bit-exact on k0-aligned plane bands against the float32 oracle run
    on the band plus its k0 - 1 halo planes (the band's windows never see the
    sub-array's end), and BDBSC against float64 (total - BDBS) with the
    BDBSC contract (S = sum|A|).
* C4 in full (round 2): every one of the 1024 planes of the box-complement
  output against the float64 decomposition; BDBS bit-exact against the float32
  oracle on the whole array; BDBSC on the whole array against float64
  total - BDBS.
* C1 (float64 1024^2 uniform [0,1), box 32^2): all three routes against the
  oracle at full size (BDBS bit-exact).
* The C4 kernels on the default path (no EXSUM_* knobs) at (64, 96, 1024),
  box 16^3, against the oracle: axis_stream<+R> + the strong fused row round
  for box-complement, axis_stream<+total> + fused pair for BDBSC, BDBS
  bit-exact.
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc
from parity import compare, depth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _bench_input(cfg, shape=None):
    import bench

    return bench.make_input(cfg, "cuda", seed=0, shape=shape)


C4_BANDS = [(0, 32), (496, 32), (992, 32)]  # (first plane, planes), k0-aligned


def _planes(t, bands):
    import torch

    return torch.cat([t[p0:p0 + m] for p0, m in bands]).cpu().numpy()


def test_c4_box_complement_full_size(ex):
    import torch

    assert not os.environ.get("EXSUM_L2PIPE")
    x = _bench_input("c4")
    n0 = x.shape[0]
    k = (16, 16, 16)
    bc = ex.box_complement_excluded(ex.Tensor(ex.Float32AddOps(), x), k).data
    got = _planes(bc, C4_BANDS)
    del bc
    xh = x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    want_x0 = [p0 + i for p0, m in C4_BANDS for i in range(m)]
    need_p = set(want_x0)                                   # P[x0-1] = sum_{y<x0}
    need_s = {x0 + k[0] for x0 in want_x0 if x0 + k[0] < n0}  # S[x0+k0] = sum_{y>=x0+k0}
    plane = np.zeros(xh.shape[1:], np.float64)
    pre, suf = {}, {}
    for y in range(n0):  # forward: sequential fold, plane by plane
        if y in need_p:
            pre[y] = plane.copy()
        plane += xh[y]
    r1 = plane  # column sums of A over axis 0
    plane = np.zeros(xh.shape[1:], np.float64)
    for y in range(n0 - 1, -1, -1):
        plane += xh[y]
        if y in need_s:
            suf[y] = plane.copy()
    del xh
    tail = orc.box_complement_excluded(r1, k[1:])
    D = depth("box-complement", (n0,) + r1.shape, k)
    worst = 0.0
    for i, x0 in enumerate(want_x0):
        s = pre[x0] + suf[x0 + k[0]] if x0 + k[0] < n0 else pre[x0]
        want = orc.bdbs_included(s, k[1:]) + tail
        err = np.abs(got[i].astype(np.float64) - want)
        ratio = float(np.max(err / (D * 2.0**-24 * want + np.finfo(np.float64).tiny)))
        worst = max(worst, ratio)
        assert ratio <= 1.0, (x0, ratio, float(np.max(err / want)))
    print(f"C4 box-complement: worst err/tol {worst:.3g} over {len(want_x0)} planes")


def test_c4_bdbs_bdbsc_full_size(ex):
    import torch

    x = _bench_input("c4")
    k = (16, 16, 16)
    t = ex.Tensor(ex.Float32AddOps(), x)
    inc = _planes(ex.bdbs_included(t, k).data, C4_BANDS)
    exc = _planes(ex.bdbs_excluded(t, k).data, C4_BANDS)
    total = float(x.double().sum())  # the check's own float64 total
    sum_abs = total                   # A >= 0
    bands = [x[p0:p0 + m + k[0] - 1].cpu().numpy() for p0, m in C4_BANDS]
    del t, x
    torch.cuda.empty_cache()
    D = depth("bdbsc", (1024,) * 3, k)
    off = 0
    for (p0, m), band in zip(C4_BANDS, bands):
        want = orc.bdbs_included(band, k)[:m]
        assert np.array_equal(inc[off:off + m].view(np.uint32), want.view(np.uint32)), p0
        want64 = total - orc.bdbs_included(band.astype(np.float64), k)[:m]
        err = np.abs(exc[off:off + m].astype(np.float64) - want64)
        assert float(err.max()) <= D * 2.0**-24 * sum_abs, (p0, float(err.max()))
        off += m


def test_c1_full_size(ex):
    import torch

    x = _bench_input("c1")
    k = (32, 32)
    a = x.cpu().numpy()
    t = ex.Tensor(ex.FloatAddOps(), x)
    got = ex.bdbs_included(t, k).data.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), orc.bdbs_included(a, k).view(np.uint64))
    for route, fn in (("bdbsc", ex.bdbs_excluded), ("box-complement", ex.box_complement_excluded)):
        got = fn(t, k).data.cpu().numpy()
        ok, ratio, rel = compare(route, got, orc.ROUTES[route](a, k, "add"), a, k, orc)
        assert ok, (route, ratio, rel)
    # the reference's own generator for add-f64 (bench.py:107-108) as well
    a = np.random.default_rng(0).random((1024, 1024))
    got = ex.bdbs_included(ex.Tensor(ex.FloatAddOps(), torch.from_numpy(a).cuda()), k).data
    assert np.array_equal(got.cpu().numpy().view(np.uint64), orc.bdbs_included(a, k).view(np.uint64))


@pytest.mark.parametrize("route", ["box-complement", "bdbsc", "bdbs"])
def test_c4_kernels_default_path(ex, route):
    assert not os.environ.get("EXSUM_L2PIPE")
    x = _bench_input("c4", shape=(64, 96, 1024))
    a = x.cpu().numpy()
    k = (16, 16, 16)
    fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
          "box-complement": ex.box_complement_excluded}[route]
    got = fn(ex.Tensor(ex.Float32AddOps(), x), k).data.cpu().numpy()
    if route == "bdbs":
        assert np.array_equal(got.view(np.uint32), orc.bdbs_included(a, k).view(np.uint32))
        return
    want = orc.ROUTES[route](a.astype(np.float64), k, "add")
    ok, ratio, rel = compare(route, got, want, a, k, orc)
    assert ok, (route, ratio, rel)


def test_c4_box_complement_every_plane(ex):
    """The headline output checked in full: every one of the 1024 planes of the
    C4 box-complement (bench.py's seeded input) against the float64 reference
    decomposition (excluded.py:129-159 peeling axis 0, see the module
    docstring), with the box-complement contract (S = BC(|A|) = the float64
    answer, A >= 0).  Prefix planes P_y = sum_{y' < y} A stream in float64; the
    suffix S_{x0+k0} = R1 - P_{x0+k0} (R1 the column sums) -- the checker's own
    float64 subtraction is ~1e-16 relative, far inside the float32 bound."""
    import collections

    import torch

    assert not os.environ.get("EXSUM_L2PIPE")
    x = _bench_input("c4")
    n0 = x.shape[0]
    k = (16, 16, 16)
    bc = ex.box_complement_excluded(ex.Tensor(ex.Float32AddOps(), x), k).data
    xh = x.cpu().numpy()
    del x
    r1 = np.zeros(xh.shape[1:], np.float64)
    for y in range(n0):
        r1 += xh[y]
    tail = orc.box_complement_excluded(r1, k[1:])
    D = depth("box-complement", (n0,) + r1.shape, k)
    tiny = np.finfo(np.float64).tiny
    ring = collections.deque()  # (index y, P_y) for the last k0 + 1 prefixes
    P = np.zeros(xh.shape[1:], np.float64)
    worst = 0.0

    def check(x0, p_x0, p_far):
        nonlocal worst
        s = p_x0 + (r1 - p_far) if p_far is not None else p_x0
        want = orc.bdbs_included(s, k[1:]) + tail
        got = bc[x0].cpu().numpy().astype(np.float64)
        ratio = float(np.max(np.abs(got - want) / (D * 2.0**-24 * want + tiny)))
        worst = max(worst, ratio)
        assert ratio <= 1.0, (x0, ratio)

    for y in range(n0 + 1):  # P holds P_y = sum of planes < y
        ring.append((y, P.copy()))
        if len(ring) > k[0] + 1:
            ring.popleft()
        x0 = y - k[0]  # output plane whose far suffix starts at y
        if x0 >= 0 and y < n0:
            check(x0, ring[0][1], P)
        if y < n0:
            P += xh[y]
    for x0 in range(max(0, n0 - k[0]), n0):  # windows reaching the end: no far suffix
        # P_{x0} from the end of the ring (the ring holds P_{n0-k0} .. P_{n0})
        p_x0 = next(p for yy, p in ring if yy == x0)
        check(x0, p_x0, None)
    del bc
    torch.cuda.empty_cache()
    print(f"C4 box-complement, all {n0} planes: worst err/tol {worst:.3g}")


def test_c4_bdbs_whole_array_bit_exact(ex):
    """C4 BDBS (float32, 1024^3, box 16^3) on bench.py's seeded input against
    the float32 C oracle (the reference's association) on the whole array: every
    element bit-identical."""
    import torch

    x = _bench_input("c4")
    k = (16, 16, 16)
    got = ex.bdbs_included(ex.Tensor(ex.Float32AddOps(), x), k).data.cpu().numpy()
    a = x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    want = orc.bdbs_included(a, k)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_c4_bdbsc_whole_array(ex):
    """C4 BDBSC on the whole array: total - BDBS in float64 on the upcast input
    (the reference algorithm, excluded.py:72-75, 88-90) within the BDBSC
    contract |got - want| <= D u sum|A|."""
    import torch

    x = _bench_input("c4")
    k = (16, 16, 16)
    got = ex.bdbs_excluded(ex.Tensor(ex.Float32AddOps(), x), k).data.cpu().numpy()
    a64 = x.cpu().numpy().astype(np.float64)
    del x
    torch.cuda.empty_cache()
    total = float(a64.sum())  # A >= 0: sum|A| = total
    want = orc.bdbs_included(a64, k)
    np.subtract(total, want, out=want)
    D = depth("bdbsc", a64.shape, k)
    del a64
    err = float(np.max(np.abs(got.astype(np.float64) - want)))
    assert err <= D * 2.0**-24 * total, (err, D * 2.0**-24 * total)
