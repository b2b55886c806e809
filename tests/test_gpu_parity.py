"""GPU parity: the CUDA path (through the C ABI) against the reference.

Every test here runs the product kernels on cuda:0 and checks them against
(1) golden vectors produced by the reference itself, and (2) the CPU oracle
(oracle/, pinned bit-exact to the reference by tests/test_oracle.py) on the
same seeded inputs, with the exactness contract in tests/parity.py.
"""

import numpy as np
import pytest

from golden_data import MONO_DTYPE, MONO_OP, load, medium_cases, small_cases
from oracle import oracle as orc
from parity import compare, float64_oracle

pytestmark = pytest.mark.gpu

ROUTE_NAMES = ("bdbs", "bdbsc", "box-complement")


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()  # fails loudly if the extension is missing
    return ex


def _mono(ex, name):
    return ex.resolve_monoid(name)


def _gpu(ex, route, mono_name, arr, box):
    import torch

    ops = _mono(ex, mono_name)
    t = ex.Tensor(ops, torch.from_numpy(np.ascontiguousarray(arr)).cuda())
    fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
          "box-complement": ex.box_complement_excluded}[route]
    out = fn(t, box)
    assert out.data.is_cuda
    return out.data.cpu().numpy()


def _check(route, mono, got, want, a, box):
    k = tuple(min(b, n) for b, n in zip(box, a.shape))
    ok, ratio, rel = compare(route, got, want, a, k, orc)
    assert ok, (route, mono, a.shape, box, ratio, rel)


def test_worked_example(ex):
    z = load("kat")
    a, box = z["worked/in"], tuple(z["worked/box"])
    assert np.array_equal(_gpu(ex, "bdbs", "add-i64", a, box), z["worked/bdbs"])
    assert np.array_equal(_gpu(ex, "bdbsc", "add-i64", a, box), z["worked/bdbsc"])
    assert np.array_equal(_gpu(ex, "box-complement", "add-i64", a, box), z["worked/box-complement"])
    assert np.array_equal(_gpu(ex, "box-complement", "max-i64", a, box),
                          z["worked/box-complement-max"])
    assert np.array_equal(_gpu(ex, "bdbs", "max-i64", a, box), z["worked/bdbs-max"])


def test_bdbs_1d_kats(ex):
    z = load("kat")
    assert ex.bdbs_1d(ex.IntAddOps(), list(range(1, 9)), 4).tolist() == [10, 14, 18, 22, 26, 21, 15, 8]
    off = 0
    for n, k in zip(z["ex1d/n"], z["ex1d/k"]):
        vals = z["ex1d/in"][off:off + n]
        assert np.array_equal(ex.bdbs_1d(ex.IntAddOps(), vals, int(k)), z["ex1d/add"][off:off + n])
        assert np.array_equal(ex.bdbs_1d(ex.IntMaxOps(), vals, int(k)), z["ex1d/max"][off:off + n])
        off += n


def test_small_golden_all_routes(ex):
    """130 reference-generated instances x 4 monoids x 3 routes."""
    n = 0
    for ci, ext, box, ins, outs in small_cases():
        for key, want in outs.items():
            parts = key.split("/")
            if len(parts) != 2 or parts[1] not in ROUTE_NAMES:
                continue
            mono, route = parts
            a = ins[mono].reshape(ext)
            got = _gpu(ex, route, mono, a, box)
            if MONO_OP[mono] == "add" and a.dtype.kind == "f" and route != "bdbs":
                # float weak/strong excluded: tolerance vs float64 evaluation
                _check(route, mono, got, float64_oracle(route, a, box, orc), a, box)
            else:
                assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (ci, key, ext, box)
            n += 1
        for mono in ("add-i64", "max-i64"):
            a = ins[mono].reshape(ext)
            assert np.array_equal(_gpu(ex, "bdbs", mono, a, box).reshape(-1), outs[f"{mono}/oracle_inc"])
            assert np.array_equal(_gpu(ex, "box-complement", mono, a, box).reshape(-1),
                                  outs[f"{mono}/oracle_exc"])
    assert n >= 1000


def test_medium_golden(ex):
    for m in medium_cases():
        a, box, route, mono = m["in"], tuple(m["box"]), m["route"], m["mono"]
        got = _gpu(ex, route, mono, a, box)
        if a.dtype.kind == "f" and route != "bdbs":
            _check(route, mono, got, float64_oracle(route, a, box, orc), a, box)
        else:
            assert np.array_equal(got.view(np.uint8), m["out"].view(np.uint8)), m["key"]


# -- random shapes vs the oracle, covering every kernel path -------------------

EDGE_SHAPES = [
    # (extents, box) -- rows/strided, k in every bucket, tails, k >= n, n == 1
    ((1,), (1,)), ((1,), (5,)), ((7,), (3,)), ((33,), (32,)), ((100,), (7,)),
    ((1000,), (37,)), ((1000,), (1000,)), ((2500,), (600,)), ((4096,), (3,)),
    ((1, 1), (2, 2)), ((3, 1), (2, 5)), ((1, 9), (3, 4)), ((17, 33), (5, 6)),
    ((64, 96), (32, 32)), ((300, 40), (100, 7)), ((40, 300), (7, 100)),
    ((130, 77), (128, 4)), ((9, 2100), (2, 1100)), ((2049, 3), (16, 2)),
    ((6, 7, 8), (2, 3, 4)), ((16, 16, 16), (4, 4, 4)), ((12, 10, 1024), (5, 3, 512)),
    ((64, 4, 3), (40, 2, 2)), ((5, 6, 7, 5, 6), (4, 4, 4, 4, 4)),
    ((4, 4, 4, 4, 4, 4), (4, 4, 4, 4, 4, 4)), ((3, 5, 2, 7), (1, 1, 1, 1)),
    ((2, 3, 130, 5), (2, 2, 64, 3)),
    # fused last-two-axes kernel (rows of 256/512/1024, unit tails, segments)
    ((3, 37, 256), (5, 8, 8)), ((2, 70, 512), (1, 2, 2)), ((2, 70, 512), (3, 16, 16)),
    ((2, 45, 1024), (2, 16, 16)), ((3, 20, 256), (2, 4, 3)), ((1, 300, 256), (1, 4, 4)),
    ((1, 130, 1024), (1, 4, 4)), ((2, 19, 512), (1, 8, 5)),
]


def _rand(rng, shape, mono):
    dt = MONO_DTYPE[mono]
    if dt == np.int64:
        return rng.integers(-2**20, 2**20, size=shape, dtype=np.int64)
    return rng.standard_normal(shape).astype(dt)


@pytest.mark.parametrize("shape,box", EDGE_SHAPES, ids=lambda v: "x".join(map(str, v)))
def test_edge_shapes_vs_oracle(ex, shape, box):
    rng = np.random.default_rng(hash((shape, box)) % 2**32)
    for mono in ("add-i64", "max-i64", "add-f64", "add-f32"):
        a = _rand(rng, shape, mono)
        for route in ROUTE_NAMES:
            if route == "bdbsc" and mono == "max-i64":
                continue
            got = _gpu(ex, route, mono, a, box)
            if a.dtype.kind == "f" and route != "bdbs":
                want = float64_oracle(route, a, box, orc)
            else:
                want = orc.ROUTES[route](a, box, MONO_OP[mono])
            _check(route, mono, got, want, a, box)


def test_int64_wraparound(ex):
    a = np.full((8, 9), 2**62, dtype=np.int64)
    a[::2] = -(2**62) - 12345
    for route in ROUTE_NAMES:
        got = _gpu(ex, route, "add-i64", a, (3, 4))
        assert np.array_equal(got, orc.ROUTES[route](a, (3, 4), "add")), route


def test_max_identity_and_negatives(ex):
    a = np.full((5, 6), np.iinfo(np.int64).min, dtype=np.int64)
    a[2, 3] = -5
    for route in ("bdbs", "box-complement"):
        assert np.array_equal(_gpu(ex, route, "max-i64", a, (2, 2)),
                              orc.ROUTES[route](a, (2, 2), "max"))
    # box covering the domain: excluded sum at the origin is the identity
    out = _gpu(ex, "box-complement", "max-i64", a, (5, 6))
    assert out[0, 0] == np.iinfo(np.int64).min


def test_unit_box_is_identity_map(ex):
    rng = np.random.default_rng(1)
    a = rng.standard_normal((7, 9))
    assert np.array_equal(_gpu(ex, "bdbs", "add-f64", a, (1, 1)), a)


def test_host_numpy_path_and_reference_tensor_class(ex):
    """numpy data goes through exsum_run_host; result keeps the caller's class/ops."""
    rng = np.random.default_rng(3)
    a = rng.integers(0, 100, size=(20, 30)).astype(np.int64)
    t = ex.Tensor(ex.IntAddOps(), a)
    for fn, route in ((ex.bdbs_included, "bdbs"), (ex.bdbs_excluded, "bdbsc"),
                      (ex.box_complement_excluded, "box-complement")):
        out = fn(t, (4, 5))
        assert type(out) is ex.Tensor and out.ops is t.ops
        assert np.array_equal(out.data, orc.ROUTES[route](a, (4, 5)))
    assert np.array_equal(t.data, a)  # input untouched


def test_windowed_sum_axis_in_place(ex):
    rng = np.random.default_rng(4)
    a = rng.integers(-9, 9, size=(6, 10, 5)).astype(np.int64)
    v = a.copy()
    ex.windowed_sum_axis(ex.IntAddOps(), v, 3, 1)
    assert np.array_equal(v, orc.windowed_pass(a, 1, 3))


# -- BASELINE-config shapes at full size (size-independent properties + oracle) --

def test_c2_full_size_int64(ex):
    """C2: 256^3 int64 in [-2^20, 2^20), box 8^3: max box-complement and + BDBSC,
    bit-exact against the oracle; + box-complement == + BDBSC exactly."""
    import torch

    rng = np.random.default_rng(0)
    a = rng.integers(-2**20, 2**20, size=(256, 256, 256), dtype=np.int64)
    box = (8, 8, 8)
    got_bc_max = _gpu(ex, "box-complement", "max-i64", a, box)
    assert np.array_equal(got_bc_max, orc.box_complement_excluded(a, box, "max"))
    got_bdbsc = _gpu(ex, "bdbsc", "add-i64", a, box)
    assert np.array_equal(got_bdbsc, orc.bdbs_excluded(a, box, "add"))
    got_bc_add = _gpu(ex, "box-complement", "add-i64", a, box)
    assert np.array_equal(got_bc_add, got_bdbsc)
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape", [(4096, 4096), (256, 256, 256), (64, 64, 64, 64),
                                   (28, 28, 28, 28, 28), (16,) * 6])
def test_c3_dimension_sweep(ex, shape):
    """C3: N ~ 2^24, k = 4 everywhere: f32 + BDBS and i64 max BDBS bit-exact."""
    rng = np.random.default_rng(0)
    box = (4,) * len(shape)
    a = rng.standard_normal(shape, dtype=np.float32)
    assert np.array_equal(_gpu(ex, "bdbs", "add-f32", a, box).view(np.uint32),
                          orc.bdbs_included(a, box).view(np.uint32))
    b = rng.integers(-2**20, 2**20, size=shape, dtype=np.int64)
    assert np.array_equal(_gpu(ex, "bdbs", "max-i64", b, box), orc.bdbs_included(b, box, "max"))


def test_c3_padded_28_to_32(ex):
    """C3's 28^5 identity-padded to 32^5 gives the 28^5 result on the crop."""
    import torch

    rng = np.random.default_rng(0)
    a = rng.standard_normal((28,) * 5, dtype=np.float32)
    t = ex.Tensor(ex.Float32AddOps(), torch.from_numpy(a).cuda())
    padded, ext = ex.pad_to_box_multiple(t, (4,) * 5)
    assert padded.extents == (28,) * 5  # 28 is already a multiple of 4
    t32 = ex.Tensor(ex.Float32AddOps(), torch.zeros((32,) * 5, dtype=torch.float32, device="cuda"))
    t32.data[(slice(0, 28),) * 5] = t.data
    out32 = ex.bdbs_included(t32, (4,) * 5)
    crop = ex.crop_to(out32, (28,) * 5)
    # identity padding only adds zeros past the boundary: equal to the 28^5 result
    want = orc.bdbs_included(a, (4,) * 5)
    np.testing.assert_array_equal(crop.data.cpu().numpy(), want)


@pytest.mark.parametrize("box", [(2, 2, 2), (8, 8, 8), (32, 32, 32), (128, 4, 1), (1, 1, 512)])
def test_c5_box_sweep(ex, box):
    """C5: 512^3 f64 standard normal: BDBS bit-exact, BDBSC within tolerance."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal((512, 512, 512))
    got = _gpu(ex, "bdbs", "add-f64", a, box)
    want = orc.bdbs_included(a, box)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    got_c = _gpu(ex, "bdbsc", "add-f64", a, box)
    # BDBSC = total - included; with included bit-exact only the total differs
    tot_tol = 1e-9 * np.abs(a).sum()
    assert np.max(np.abs(got_c - (a.sum() - want))) <= tot_tol
