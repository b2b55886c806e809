"""Balanced unit ranges of the fused pass pair and the balanced last wave of
the axis pass (csrc/fused_pair.cuh, csrc/axis_stream.cuh): on arrays of at
least four units per SM with one resident CTA per SM (1024-wide float32 rows,
512-wide 8-byte rows) a CTA's contiguous range of units is split wherever it
crosses a line, so pieces start and end mid-line.  Ragged axis lengths (the
last unit and the last window block partial), line counts that are not a
multiple of the SM count and several outer indices, against the oracle:
bit-exact for BDBS (floats too), int64 and max; the float parity bound for the
excluded routes; and identical bits with the balancing switched off.
EXSUM_FP_BALANCED=2 / EXSUM_AS_BAL_TAIL=2 take the balanced schedules wherever the
kernels allow them (not only where the cost model picks them), so the small
shapes here run them too -- pieces of a single unit, CTAs with empty ranges."""

import os

import numpy as np
import pytest

from oracle import oracle as orc
from parity import compare, float64_oracle

pytestmark = pytest.mark.gpu

CASES = [
    # monoid, extents, box
    ("add-f32", (37, 300, 1024), (16, 16, 16)),   # 37 lines x 19 units, last unit 12 rows
    ("add-f32", (41, 261, 1024), (8, 8, 8)),      # last block of axis 1 partial (261 = 32*8 + 5)
    ("add-f32", (150, 77, 1024), (4, 16, 16)),    # 150 lines of 5 units: more lines than SMs
    ("add-f64", (23, 530, 512), (8, 8, 8)),
    ("add-f64", (60, 200, 512), (2, 16, 16)),
    ("add-i64", (29, 410, 512), (16, 8, 8)),
    ("max-i64", (33, 333, 512), (3, 16, 16)),
    ("add-f32", (2, 3, 200, 1024), (2, 2, 8, 8)),  # d = 4: outer = 6 lines of 13 units ... 4-D outer
    ("add-f32", (700, 16, 1024), (16, 16, 16)),    # one unit per line
    ("add-f32", (130, 200, 1024), (16, 2, 4)),     # axis pass: 200 strips of 9 units, k < 8 pair
    ("add-f64", (70, 301, 512), (4, 4, 4)),        # axis pass: 301 strips of 5 units
    ("add-f32", (5, 40, 1024), (2, 8, 8)),         # fewer units than SMs: empty ranges
    # strips (rows longer than the widest row template): a line is one strip of one outer index
    ("add-f32", (3, 210, 3072), (2, 16, 16)),
    ("add-f32", (170, 2048), (8, 8)),
    ("add-f64", (2, 157, 1536), (2, 16, 16)),
    ("max-i64", (7, 100, 1024), (1, 16, 16)),
]


def _data(mono, shape, seed):
    rng = np.random.default_rng(seed)
    if mono.endswith("i64"):
        return rng.integers(-2**40, 2**40, size=shape, dtype=np.int64)
    dt = np.float32 if mono == "add-f32" else np.float64
    return rng.standard_normal(shape).astype(dt)


@pytest.mark.parametrize("mono,ext,box", CASES, ids=lambda v: str(v))
def test_balanced_schedules_match_the_oracle(mono, ext, box, monkeypatch):
    import torch

    import paper_2106_00124_b200 as ex

    ops = ex.resolve_monoid(mono)
    a = _data(mono, ext, seed=sum(ext))
    x = torch.from_numpy(a).cuda()
    op = "max" if mono == "max-i64" else "add"
    routes = ["bdbs", "box-complement"] + (["bdbsc"] if ops.has_inverse else [])
    fns = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
           "box-complement": ex.box_complement_excluded}
    for route in routes:
        monkeypatch.setenv("EXSUM_FP_BALANCED", "2")
        monkeypatch.setenv("EXSUM_AS_BAL_TAIL", "2")
        got = fns[route](ex.Tensor(ops, x), box).data.cpu().numpy()
        monkeypatch.delenv("EXSUM_FP_BALANCED")
        monkeypatch.delenv("EXSUM_AS_BAL_TAIL")
        auto = fns[route](ex.Tensor(ops, x), box).data.cpu().numpy()  # the cost model's choice
        assert np.array_equal(got.view(np.uint8), auto.view(np.uint8)), route
        if route == "bdbs" or a.dtype.kind == "i":
            want = orc.ROUTES[route](a, box, op)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), route
        else:
            k = tuple(min(b, n) for b, n in zip(box, ext))
            ok, ratio, rel = compare(route, got, float64_oracle(route, a, box, orc, op), a, k, orc)
            assert ok, (route, ratio, rel)
        # the uniform schedules give the same bits (only the work split differs)
        monkeypatch.setenv("EXSUM_FP_BALANCED", "0")
        monkeypatch.setenv("EXSUM_AS_BAL_TAIL", "0")
        plain = fns[route](ex.Tensor(ops, x), box).data.cpu().numpy()
        monkeypatch.delenv("EXSUM_FP_BALANCED")
        monkeypatch.delenv("EXSUM_AS_BAL_TAIL")
        assert np.array_equal(got.view(np.uint8), plain.view(np.uint8)), route


def test_balanced_schedules_random_shapes(monkeypatch):
    """Random ragged shapes on the one-CTA-per-SM row widths with the balanced
    schedules forced: every route against the schedules switched off, bit for
    bit (the uniform schedules are pinned to the oracle by the other suites),
    and BDBS against the oracle directly."""
    import torch

    import paper_2106_00124_b200 as ex

    rng = np.random.default_rng(int(os.environ.get("EXSUM_FUZZ_SEED", "2106")) + 77)
    n_cases = int(os.environ.get("EXSUM_BALANCED_CASES", "20"))
    fns = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
           "box-complement": ex.box_complement_excluded}
    for case in range(n_cases):
        mono = str(rng.choice(["add-f32", "add-f64", "add-i64", "max-i64"]))
        width = 1024 if mono == "add-f32" else 512
        n1 = int(rng.integers(3, 400))
        lead = tuple(int(v) for v in rng.integers(1, 40, size=int(rng.integers(1, 3))))
        if rng.random() < 0.3:  # many strips for the axis pass: a long axis 0 over >= 149 strips
            lead, n1 = (int(rng.integers(64, 200)),), int(rng.integers(149, 330))
        ext = lead + (n1, width)
        k = int(rng.choice([2, 4, 8, 16]))
        box = tuple(int(rng.choice([1, k, 3, n])) if rng.random() < 0.25 else k for n in ext)
        ops = ex.resolve_monoid(mono)
        a = _data(mono, ext, seed=1000 + case)
        x = torch.from_numpy(a).cuda()
        op = "max" if mono == "max-i64" else "add"
        routes = ["bdbs", "box-complement"] + (["bdbsc"] if ops.has_inverse else [])
        for route in routes:
            monkeypatch.setenv("EXSUM_FP_BALANCED", "2")
            monkeypatch.setenv("EXSUM_AS_BAL_TAIL", "2")
            forced = fns[route](ex.Tensor(ops, x), box).data.cpu().numpy()
            monkeypatch.setenv("EXSUM_FP_BALANCED", "0")
            monkeypatch.setenv("EXSUM_AS_BAL_TAIL", "0")
            plain = fns[route](ex.Tensor(ops, x), box).data.cpu().numpy()
            monkeypatch.delenv("EXSUM_FP_BALANCED")
            monkeypatch.delenv("EXSUM_AS_BAL_TAIL")
            assert np.array_equal(forced.view(np.uint8), plain.view(np.uint8)), (case, mono, ext, box, route)
            if route == "bdbs":
                want = orc.ROUTES[route](a, box, op)
                assert np.array_equal(forced.view(np.uint8), want.view(np.uint8)), (case, mono, ext, box)
