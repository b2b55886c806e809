"""Randomised sweep of every route x monoid x dtype against the oracle
(shapes d = 1..5 up to ~64 per axis, boxes including k >= n and k = 1, both
the device and the host path).  EXSUM_FUZZ_CASES sets the count (default 150;
a long run used 3000)."""

import os

import numpy as np
import pytest

from golden_data import mono_op
from oracle import oracle as orc
from parity import compare, float64_oracle

pytestmark = pytest.mark.gpu

MONOS = ["add-i64", "max-i64", "add-f64", "add-f32", "mod-add:97", "mod-add:2147483648"]
ROUTES = ["bdbs", "bdbsc", "box-complement", "sat", "satc", "corners"]


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _special_case(rng):
    """Shapes that take the shape-specialised kernels: cubic trailing blocks
    (k_block_cubic: NL 16/28/32/64), two leading axes of 16/28 (k_outer_pair)
    and rows wider than the fused pair's widest template (row strips), the
    tiled pair (window 32 on the last two axes) and the marginal form of max
    (any shape; box-complement on max-i64 takes it)."""
    kind = int(rng.integers(4))
    K = int(rng.choice([2, 4, 8]))
    if kind == 3:
        n1, n2 = int(rng.integers(32, 200)), int(rng.integers(32, 300))
        shape = (int(rng.integers(1, 5)), n1, n2) if rng.random() < 0.5 else (n1, n2)
        box = (int(rng.choice([1, 3, 32])),) * (len(shape) - 2) + (32, 32)
        return shape, box
    if kind == 0:
        nl = int(rng.choice([16, 28, 32, 64]))
        m = 3 if nl <= 28 and rng.random() < 0.5 else 2
        lead = int(rng.integers(1, max(2, 400_000 // nl ** m) + 1))
        shape = (lead,) + (nl,) * m
    elif kind == 1:
        na = int(rng.choice([16, 28]))
        inner = int(rng.choice([16, 32, 48, 64, 80]))
        shape = (int(rng.integers(1, 4)), na, na, inner) if rng.random() < 0.5 else (na, na, inner)
    else:
        w = int(rng.choice([1536, 2048, 3072, 4096]))
        shape = (int(rng.integers(1, 3)), int(rng.integers(2, 60)), w) if rng.random() < 0.4 \
            else (int(rng.integers(2, 100)), w)
    box = tuple(K if rng.random() < 0.85 else int(rng.choice([1, K, n])) for n in shape)
    return shape, box


def _case(rng):
    if rng.random() < 0.25:
        return _special_case(rng)
    d = int(rng.integers(1, 6))
    cap = {1: 4096, 2: 160, 3: 48, 4: 20, 5: 10}[d]
    shape = tuple(int(v) for v in rng.integers(1, cap + 1, size=d))
    if rng.random() < 0.3:  # widths that hit the fused / vector paths
        shape = shape[:-1] + (int(rng.choice([256, 512, 1024])),)
        if np.prod(shape) > 2_000_000:
            shape = (1,) * (d - 1) + shape[-1:]
    box = tuple(int(rng.integers(1, n + 3)) if rng.random() < 0.8 else int(rng.choice([1, 2, 4, 8, 16, 32]))
                for n in shape)
    return shape, box


def test_random_sweep(ex):
    import torch

    n_cases = int(os.environ.get("EXSUM_FUZZ_CASES", "150"))
    rng = np.random.default_rng(int(os.environ.get("EXSUM_FUZZ_SEED", "2106")))
    fns = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
           "box-complement": ex.box_complement_excluded, "sat": ex.sat_included,
           "satc": ex.sat_excluded, "corners": ex.corners_excluded}
    done = 0
    while done < n_cases:
        shape, box = _case(rng)
        mono = MONOS[int(rng.integers(len(MONOS)))]
        route = ROUTES[int(rng.integers(len(ROUTES)))]
        if mono == "max-i64" and route in ("bdbsc", "sat", "satc"):
            continue
        if route == "corners" and len(shape) not in (2, 3):
            continue
        ops = ex.Float32AddOps() if mono == "add-f32" else ex.resolve_monoid(mono)
        dt = np.dtype(ops.dtype)
        a = (rng.standard_normal(shape).astype(dt) if dt.kind == "f"
             else rng.integers(-10**6, 10**6, size=shape, dtype=np.int64))
        device = bool(rng.random() < 0.7)
        data = torch.from_numpy(a).cuda() if device else a.copy()
        got = fns[route](ex.Tensor(ops, data), box).data
        got = got.cpu().numpy() if device else got
        _check(route, mono, got, a, box, shape, ("device" if device else "host"))
        done += 1


def _medium_case(rng):
    d = int(rng.integers(2, 5))
    w = int(rng.choice([256, 512, 1024, 384, 1000, 4096, 7]))
    target = int(rng.integers(1_000_000, 8_000_000))
    rest = max(1, target // w)
    if d == 2:
        shape = (rest, w)
    elif d == 3:
        a = int(rng.integers(1, max(2, int(rest ** 0.5)) + 1))
        shape = (a, max(1, rest // a), w)
    else:
        a = int(rng.integers(1, max(2, int(rest ** (1 / 3))) + 1))
        b = int(rng.integers(1, max(2, int(rest ** (1 / 3))) + 1))
        shape = (a, b, max(1, rest // (a * b)), w)
    box = tuple(int(rng.choice([1, 2, 3, 4, 8, 16, 32, 64, n, n + 5])) for n in shape)
    return shape, box


def _check(route, mono, got, a, box, shape, tag):
    want = orc.ROUTES[route](a, box, mono_op(mono))
    if a.dtype.kind != "f" or route == "bdbs" or np.array_equal(got, want):
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (route, mono, shape, box, tag)
        return
    # floats off the bit-exact contract: the route's tolerance (corners: a
    # segmented scan reassociates; same quantity as box-complement)
    k = tuple(min(b, e) for b, e in zip(box, shape))
    r = "box-complement" if route == "corners" else route
    ok, ratio, _ = compare(r, got, float64_oracle(r, a, k, orc), a, k, orc)
    assert ok, (route, mono, shape, box, tag, ratio)


def test_random_medium_sweep(ex):
    """Sizes that reach the large-array kernels (fused pair, axis stream, TMA
    bulk, SAT chain query, segmented scans), device and host paths."""
    import torch

    n_cases = int(os.environ.get("EXSUM_FUZZ_MEDIUM", "24"))
    rng = np.random.default_rng(int(os.environ.get("EXSUM_FUZZ_SEED", "2106")) + 1)
    fns = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
           "box-complement": ex.box_complement_excluded, "sat": ex.sat_included,
           "satc": ex.sat_excluded, "corners": ex.corners_excluded}
    done = 0
    while done < n_cases:
        shape, box = _medium_case(rng)
        mono = ["add-i64", "max-i64", "mod-add:1000003", "add-f64", "add-f32"][int(rng.integers(5))]
        route = ROUTES[int(rng.integers(len(ROUTES)))]
        if mono == "max-i64" and route in ("bdbsc", "sat", "satc"):
            continue
        if route == "corners" and len(shape) not in (2, 3):
            continue
        ops = ex.Float32AddOps() if mono == "add-f32" else ex.resolve_monoid(mono)
        dt = np.dtype(ops.dtype)
        a = (rng.standard_normal(shape).astype(dt) if dt.kind == "f"
             else rng.integers(-10**9, 10**9, size=shape, dtype=np.int64))
        device = bool(rng.random() < 0.7)
        data = torch.from_numpy(a).cuda() if device else a.copy()
        got = fns[route](ex.Tensor(ops, data), box).data
        got = got.cpu().numpy() if device else np.asarray(got)
        _check(route, mono, got, a, box, shape, "device" if device else "host")
        done += 1


def test_random_large_host(ex):
    """Host calls of >= 64 MB (the pipelined single-call BDBS and the chunked
    host routes) on random shapes and boxes."""
    n_cases = int(os.environ.get("EXSUM_FUZZ_LARGE", "3"))
    rng = np.random.default_rng(int(os.environ.get("EXSUM_FUZZ_SEED", "2106")) + 2)
    for _ in range(n_cases):
        d = int(rng.integers(2, 4))
        n_last = int(rng.choice([256, 1000, 1024]))
        n0 = int(rng.integers(64, 600))
        rows = int(9_000_000 * rng.uniform(1.0, 1.6)) // n_last  # >= 9e6 elements (>= 64 MB in 8 B)
        shape = (n0, rows // n0 + 1, n_last) if d == 3 else (rows, n_last)
        box = tuple(int(rng.choice([1, 2, 5, 16, 33, n])) for n in shape)
        mono = ["add-i64", "max-i64", "add-f64"][int(rng.integers(3))]
        route = ["bdbs", "bdbs", "box-complement"][int(rng.integers(3))]
        ops = ex.resolve_monoid(mono)
        a = (rng.standard_normal(shape) if mono == "add-f64"
             else rng.integers(-10**9, 10**9, size=shape, dtype=np.int64))
        fn = ex.bdbs_included if route == "bdbs" else ex.box_complement_excluded
        got = np.asarray(fn(ex.Tensor(ops, a.copy()), box).data)
        _check(route, mono, got, a, box, shape, "host-large")
