"""GPU parity for the SURVEY 8(f) rows: the "sat" / "satc" routes
(included.py:37-121, excluded.py:83-85) and the mod-add:<m> monoid
(monoid.py:235-286) on every route, through the C ABI on cuda:0.

Pinned to golden vectors produced by the reference (tests/golden/ext.npz) and
to the CPU oracle (tests/test_oracle.py pins it to the reference) at larger
sizes.  Integer and mod-add results are bit-exact; float sat is bit-exact
where the table scans run unsegmented, otherwise within tests/parity.py.
"""

import numpy as np
import pytest

from golden_data import corner_cases, ext_cases, mono_op
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


def _fn(ex, route):
    return {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
            "box-complement": ex.box_complement_excluded, "sat": ex.sat_included,
            "satc": ex.sat_excluded, "corners": ex.corners_excluded,
            "corners-spine": ex.corners_spine_excluded}[route]


def _mono(ex, name):
    if name == "add-f32":
        return ex.Float32AddOps()
    return ex.resolve_monoid(name)


def _run(ex, route, mono, arr, box, device=True):
    import torch

    ops = _mono(ex, mono)
    arr = np.ascontiguousarray(arr)
    data = torch.from_numpy(arr).cuda() if device else arr
    out = _fn(ex, route)(ex.Tensor(ops, data), box)
    return out.data.cpu().numpy() if device else out.data


def _bits_equal(a, b):
    return a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_ext_golden_vectors(ex):
    """Every sat/satc and mod-add vector of the reference, device and host paths."""
    n = 0
    for m in ext_cases():
        route = m["route"]
        if route.startswith("oracle_"):
            continue
        box = tuple(m["box"])
        a = m["in"]
        for device in (True, False):
            got = _run(ex, route, m["mono"], a, box, device)
            if a.dtype.kind != "f" or route == "sat":
                assert _bits_equal(got, m["out"]), (m["key"], device)
            else:
                k = tuple(min(b, e) for b, e in zip(box, a.shape))
                want = float64_oracle(route, a, k, orc)
                ok, ratio, rel = compare(route, got, want, a, k, orc)
                assert ok, (m["key"], ratio, rel)
        n += 1
    assert n >= 500


def test_mod_add_matches_brute_force(ex):
    """mod-add against the reference's own brute-force oracle outputs."""
    seen = 0
    for m in ext_cases():
        if not m["route"].startswith("oracle_") or not m["mono"].startswith("mod-add:"):
            continue
        route = "bdbs" if m["route"] == "oracle_inc" else "box-complement"
        got = _run(ex, route, m["mono"], m["in"], tuple(m["box"]))
        want = m["out"]
        mod = int(m["mono"].split(":")[1])
        # the brute force starts each fold from the first raw value, so a
        # one-element box (or complement) keeps it unreduced; compare residues
        assert np.array_equal(np.mod(got, mod), np.mod(want, mod)), m["key"]
        seen += 1
    assert seen >= 40


@pytest.mark.parametrize("mod", [2, 97, 1000003, 2**31])
@pytest.mark.parametrize("route", ["bdbs", "bdbsc", "box-complement", "sat", "satc"])
def test_mod_add_random_vs_oracle(ex, route, mod):
    rng = np.random.default_rng(mod % 1000 + len(route))
    for shape, box in [((37, 41), (5, 1)), ((9, 8, 7), (3, 8, 2)), ((64, 64, 16), (4, 4, 4)),
                       ((6, 5, 4, 3), (1, 1, 1, 1)), ((1000,), (7,)), ((33, 65), (33, 3))]:
        a = rng.integers(-5 * mod, 5 * mod, size=shape, dtype=np.int64)
        a[..., ::3] = rng.integers(-2**45, 2**45, size=a[..., ::3].shape)
        want = orc.ROUTES[route](a, box, f"mod-add:{mod}")
        got = _run(ex, route, f"mod-add:{mod}", a, box)
        assert np.array_equal(got, want), (route, mod, shape, box)


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.int64])
def test_sat_medium_shapes(ex, dtype):
    rng = np.random.default_rng(11)
    for shape, box in [((256, 256, 64), (4, 4, 4)), ((96, 80), (32, 32)), ((30, 20, 10, 6), (3, 4, 5, 2)),
                       ((12,) * 5, (4,) * 5), ((8,) * 6, (2,) * 6), ((4,) * 7, (2,) * 7),
                       ((3000, 5), (17, 2)), ((5, 3000), (1, 64))]:
        if dtype == np.int64:
            a = rng.integers(-2**20, 2**20, size=shape, dtype=np.int64)
            mono = "add-i64"
        else:
            a = rng.standard_normal(shape).astype(dtype)
            mono = "add-f32" if dtype == np.float32 else "add-f64"
        for route in ("sat", "satc"):
            got = _run(ex, route, mono, a, box)
            if dtype == np.int64:
                assert np.array_equal(got, orc.ROUTES[route](a, box, "add")), (route, shape)
            elif route == "sat":
                # unsegmented scans: the reference's association, bit for bit
                assert _bits_equal(got, orc.sat_included(a, box)), (shape, box)
            else:
                k = tuple(min(b, e) for b, e in zip(box, shape))
                ok, ratio, rel = compare(route, got, float64_oracle(route, a, k, orc), a, k, orc)
                assert ok, (route, shape, ratio, rel)


@pytest.mark.parametrize("dtype", [np.float64, np.int64])
def test_sat_segmented_long_axes(ex, dtype):
    """Too few lines to fill the GPU: segmented scans (exact for int64)."""
    rng = np.random.default_rng(12)
    for shape, box in [((1 << 21,), (9,)), ((3, 1 << 19), (2, 100)), ((1 << 18, 2), (1000, 2)),
                       ((100003,), (3,))]:
        a = (rng.integers(-1000, 1000, size=shape, dtype=np.int64) if dtype == np.int64
             else rng.random(shape))
        mono = "add-i64" if dtype == np.int64 else "add-f64"
        for route in ("sat", "satc"):
            got = _run(ex, route, mono, a, box)
            want = orc.ROUTES[route](a, box, "add")
            if dtype == np.int64:
                assert np.array_equal(got, want), (route, shape)
            else:
                k = tuple(min(b, e) for b, e in zip(box, shape))
                ok, ratio, rel = compare(route, got, float64_oracle(route, a, k, orc), a, k, orc)
                assert ok, (route, shape, ratio, rel)


def test_mod_add_windowed_and_1d(ex):
    ops = ex.ModAddOps(7)
    vals = np.array([3, -9, 40, 6, 100, -1, 2], dtype=np.int64)
    for k in range(1, 9):
        want = orc.bdbs_included(vals, (k,), "mod-add:7")
        assert np.array_equal(ex.bdbs_1d(ops, vals, k), want), k
    a = np.arange(-30, 30, dtype=np.int64).reshape(6, 10) * 13
    v = a.copy()
    ex.windowed_sum_axis(ops, v, 4, 1)
    assert np.array_equal(v, orc.windowed_pass(a, 1, 4, "mod-add:7"))


def test_sat_workspace_and_launches(ex):
    import torch

    a = torch.rand(64, 64, 64, device="cuda")
    t = ex.Tensor(ex.Float32AddOps(), a)
    before = ex._native.total_launch_count()
    ex.sat_included(t, (4, 4, 4))
    torch.cuda.synchronize()
    assert ex._native.total_launch_count() - before == 4  # 3 scans + 1 query


def test_corners_golden_vectors(ex):
    """corners / corners-spine (excluded.py:191-292) against the reference:
    sequential scans and the reference's accumulation order, so floats too are
    bit-exact."""
    n = 0
    for m in corner_cases():
        for route in ("corners", "corners-spine"):
            for device in (True, False):
                got = _run(ex, route, m["mono"], m["in"], tuple(m["box"]), device)
                assert _bits_equal(got, m["out"]), (m["tag"], route, device)
        n += 1
    assert n >= 50


@pytest.mark.parametrize("mono", ["add-i64", "max-i64", "add-f64", "add-f32", "mod-add:97"])
def test_corners_vs_oracle_and_box_complement(ex, mono):
    rng = np.random.default_rng(7)
    for shape, box in [((200, 150), (9, 30)), ((64, 48, 80), (4, 7, 16)), ((1, 300), (1, 5)),
                       ((5000, 3), (100, 2)), ((3, 4, 5000), (2, 2, 64))]:
        if mono.startswith("add-f"):
            a = rng.random(shape).astype(np.float32 if mono == "add-f32" else np.float64)
        else:
            a = rng.integers(-2**20, 2**20, size=shape, dtype=np.int64)
        got = _run(ex, "corners", mono, a, box)
        want = orc.corners_excluded(a, box, mono_op(mono))
        if a.dtype.kind == "f" and max(shape) < 4096:
            assert _bits_equal(got, want), (mono, shape)  # unsegmented scans: exact
        elif a.dtype.kind == "f":
            k = tuple(min(b, e) for b, e in zip(box, shape))
            ok, ratio, rel = compare("box-complement", got,
                                     orc.corners_excluded(a.astype(np.float64), box), a, k, orc)
            assert ok, (mono, shape, ratio)
        else:
            assert np.array_equal(got, want), (mono, shape)
            # and the strong excluded sum is the same whichever decomposition
            assert np.array_equal(got, _run(ex, "box-complement", mono, a, box))


def test_run_many_host_batch_matches_single_calls(ex):
    """exsum_route_host_batch: pipelined copies, same results as one call each."""
    rng = np.random.default_rng(21)
    for algo, mono, shape, box in [("box-complement", "add-f32", (40, 33, 256), (4, 3, 16)),
                                   ("bdbsc", "add-i64", (17, 64, 9), (3, 8, 2)),
                                   ("sat", "mod-add:97", (30, 40), (5, 7)),
                                   ("bdbs", "max-i64", (1000,), (33,)),
                                   ("corners", "add-f64", (20, 30), (4, 5))]:
        ops = _mono(ex, mono)
        arrs = []
        for _ in range(5):
            if mono.startswith("add-f"):
                a = rng.random(shape).astype(ops.dtype)
            else:
                a = rng.integers(-1000, 1000, size=shape, dtype=np.int64)
            arrs.append(ex.Tensor(ops, a))
        outs = ex.run_many(algo, arrs, box)
        for t, o in zip(arrs, outs):
            want = _fn(ex, algo)(t, box).data
            assert _bits_equal(np.asarray(o.data), np.asarray(want)), algo
    with pytest.raises(ex.UsageError):
        ex.run_many("bdbs", [ex.Tensor(ex.IntAddOps(), np.zeros((3, 4), dtype=np.int64)),
                             ex.Tensor(ex.IntAddOps(), np.zeros((4, 3), dtype=np.int64))], (2, 2))


@pytest.mark.parametrize("d", [7, 9, 12])
def test_high_dimensional_routes(ex, d):
    """d up to 12 (the generic kernels: box-complement's recursive tail, the
    2^d-term SAT query), every dtype/operator, against the oracle."""
    rng = np.random.default_rng(40 + d)
    shape = tuple(int(v) for v in rng.integers(1, 4, size=d))
    while int(np.prod(shape)) < 64:
        shape = tuple(int(v) for v in rng.integers(1, 4, size=d))
    box = tuple(int(v) for v in rng.integers(1, 4, size=d))
    for mono in ("add-i64", "max-i64", "add-f64", "mod-add:13"):
        a = (rng.standard_normal(shape) if mono == "add-f64"
             else rng.integers(-50, 50, size=shape, dtype=np.int64))
        op = mono_op(mono)
        routes = ["bdbs", "box-complement"] + ([] if mono == "max-i64" else ["bdbsc", "sat", "satc"])
        for route in routes:
            got = _run(ex, route, mono, a, box)
            want = orc.ROUTES[route](a, box, op)
            if a.dtype.kind == "f" and route != "bdbs" and route != "sat":
                k = tuple(min(b, e) for b, e in zip(box, shape))
                ok, ratio, rel = compare(route, got, float64_oracle(route, a, k, orc), a, k, orc)
                assert ok, (d, route, ratio)
            else:
                assert _bits_equal(got, want), (d, mono, route, shape, box)


@pytest.mark.parametrize("shape,box,dt", [
    ((520, 130, 256), (16, 4, 8), np.float32),      # 69 MB, uneven chunks
    ((300, 256, 128), (8, 8, 8), np.float64),       # 78 MB
    ((1000, 8192), (33, 5), np.int64),              # 65 MB, d = 2, k0 not a power of 2
    ((257, 256, 256), (1, 4, 4), np.float32),       # k0 = 1: no axis-0 stage
    ((129, 256, 512), (100, 3, 2), np.int64),       # max, window close to the extent
])
def test_host_bdbs_pipelined_is_exact(ex, shape, box, dt):
    """Numpy-in/numpy-out BDBS >= 64 MB runs pipelined over axis-0 chunks
    (H2D / compute / D2H overlapped); bit-identical to the oracle."""
    rng = np.random.default_rng(sum(shape))
    if np.dtype(dt).kind == "f":
        a = rng.standard_normal(shape).astype(dt)
        mono = "add-f32" if dt == np.float32 else "add-f64"
        op = "add"
    else:
        a = rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)
        mono, op = ("max-i64", "max") if box[0] == 100 else ("add-i64", "add")
    got = _run(ex, "bdbs", mono, a, box, device=False)
    want = orc.bdbs_included(a, box, op)
    assert _bits_equal(got, want), (shape, box, mono)
