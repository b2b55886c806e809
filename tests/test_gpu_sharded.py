"""Sharded stages on one GPU: virtual ranks (sharded.run_loopback) drive the
C-ABI stage entry points (exsum_shard_axis0_pass, exsum_bdbs_finish,
exsum_box_complement_finish) through the real slab arithmetic; results must
equal the single-GPU route bit for bit (integers, float BDBS) or satisfy the
float parity contract (BDBSC totals and box-complement row reductions are
reassociated per shard)."""

import numpy as np
import pytest

from oracle import oracle as orc
from parity import compare, float64_oracle

pytestmark = pytest.mark.gpu

CASES = [
    # extents, box, monoid, world
    ((64, 96, 256), (8, 8, 8), "add-f32", 4),
    ((64, 96, 256), (8, 8, 8), "max-i64", 3),
    ((37, 20, 28), (4, 3, 5), "add-i64", 3),
    ((50, 40), (16, 7), "add-f64", 3),           # d = 2
    ((45, 12, 32), (20, 4, 4), "add-f64", 2),    # k0 = 20: fallback pass into a temporary
    ((9, 30, 1024), (2, 16, 16), "add-f32", 4),  # fused kernels on the shard
    ((5, 8, 8), (8, 2, 2), "add-i64", 2),        # one empty rank
]


@pytest.mark.parametrize("ext,box,mono,world", CASES, ids=lambda v: str(v))
def test_loopback_matches_single_gpu(ext, box, mono, world):
    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200.sharded import CudaEngine, run_loopback

    ops = ex.resolve_monoid(mono)
    rng = np.random.default_rng(7)
    if ops.dtype.kind == "i":
        a = rng.integers(-2**20, 2**20, size=ext, dtype=np.int64)
    else:
        a = rng.standard_normal(ext).astype(ops.dtype)
    x = torch.from_numpy(a).cuda()
    engine = CudaEngine(ops, x.device)
    routes = ["bdbs", "box-complement"] + (["bdbsc"] if ops.has_inverse else [])
    for route in routes:
        fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
              "box-complement": ex.box_complement_excluded}[route]
        single = fn(ex.Tensor(ops, x), box).data.cpu().numpy()
        sharded = run_loopback(route, ops, x, box, world, engine).cpu().numpy()
        plain = run_loopback(route, ops, x, box, world, engine, split=False).cpu().numpy()
        assert sharded.shape == single.shape
        if route != "bdbsc":  # the split only regroups the per-rank total
            assert np.array_equal(sharded.view(np.uint8), plain.view(np.uint8)), route
        if route != "bdbs" and ops.dtype.kind == "f":
            # reassociated float totals / row reductions: the parity contract
            k = tuple(min(b, n) for b, n in zip(box, ext))
            ok, ratio, rel = compare(route, sharded, float64_oracle(route, a, box, orc), a, k, orc)
            assert ok, (route, ratio, rel)
        else:
            assert np.array_equal(sharded.view(np.uint8), single.view(np.uint8)), route
        if ops.dtype.kind == "i":
            op = "max" if mono == "max-i64" else "add"
            assert np.array_equal(sharded, orc.ROUTES[route](a, box, op)), route
