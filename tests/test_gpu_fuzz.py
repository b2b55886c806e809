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


def _case(rng):
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
        op = mono_op(mono)
        if dt.kind != "f":
            want = orc.ROUTES[route](a, box, op)
            assert np.array_equal(got, want), (route, mono, shape, box, device)
        else:
            k = tuple(min(b, e) for b, e in zip(box, shape))
            if route in ("bdbs", "corners"):
                want = orc.ROUTES[route](a, box, op)
                assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), \
                    (route, mono, shape, box, device)
            else:
                ok, ratio, rel = compare(route, got, float64_oracle(route, a, k, orc), a, k, orc)
                assert ok, (route, mono, shape, box, device, ratio)
        done += 1
