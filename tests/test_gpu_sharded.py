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
    ((5, 8, 8), (8, 2, 2), "max-i64", 2),        # marginal form with an empty rank
    ((33, 17, 66), (4, 5, 8), "max-i64", 4),     # marginal form, uneven slabs, odd rows
    # the own-rows tail (exsum_shard_bc_tail) on uneven slabs, k1 = n1, k1 = 1, one
    # block along axis 0 (a single non-empty rank), more ranks than blocks
    ((33, 17, 66), (4, 5, 8), "add-i64", 4),
    ((40, 7, 19), (3, 7, 2), "add-f64", 5),
    ((16, 16, 16), (16, 1, 4), "add-i64", 2),
    ((130, 33, 40), (8, 33, 5), "add-i64", 8),
    ((12, 260, 24), (5, 9, 3), "add-f32", 6),
    ((1024, 64, 32), (16, 16, 16), "add-f32", 8),
]


def test_sharded_max_takes_the_marginal_form():
    """Box-complement over max shards as per-axis marginals: no halo, an
    all-reduce of sum(ext) values (csrc/idem_max.cu)."""
    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200.sharded import CudaEngine, ShardedRunner, run_loopback

    ops = ex.IntMaxOps()
    ext, box = (40, 24, 48), (8, 4, 8)
    engine = CudaEngine(ops, torch.device("cuda"))
    r = ShardedRunner("box-complement", ops, ext, box, 1, 3, torch.device("cuda"),
                      comm=object(), engine=engine)
    assert r.idem
    a = np.random.default_rng(1).integers(-2**40, 2**40, size=ext, dtype=np.int64)
    got = run_loopback("box-complement", ops, torch.from_numpy(a).cuda(), box, 3, engine)
    assert np.array_equal(got.cpu().numpy(), orc.box_complement_excluded(a, box, "max"))


def test_sharded_3d_box_complement_takes_the_own_rows_tail():
    """A 3-D box-complement over + computes only its own rows of the tail on
    every rank (exsum_shard_bc_tail: R2 all-gathered, R's halo rows exchanged)
    -- the route the loopback cases below must be exercising."""
    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200.sharded import CudaEngine, ShardedRunner

    dev = torch.device("cuda")
    for mono, ext, box in (("add-i64", (37, 20, 28), (4, 3, 5)), ("add-f32", (64, 96, 256), (8, 8, 8)),
                           ("add-f32", (1024, 1024, 1024), (16, 16, 16)), ("add-f64", (45, 12, 32), (20, 4, 4))):
        ops = ex.resolve_monoid(mono)
        r = ShardedRunner("box-complement", ops, ext, box, 1, 3, dev, comm=object(),
                          engine=CudaEngine(ops, dev))
        assert r.own_tail and not r.idem, (mono, ext)
    ops = ex.resolve_monoid("add-f64")  # d = 2: R is 1-D, the tail is all-gathered
    r = ShardedRunner("box-complement", ops, (50, 40), (16, 7), 1, 3, dev, comm=object(),
                      engine=CudaEngine(ops, dev))
    assert not r.own_tail


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


def _nccl_world1_worker(port, q):
    """One process, NCCL process group of world size 1 on cuda:0: the real
    DistComm (NCCL all-gathers, rank-order totals) and CudaEngine stages."""
    import os
    import sys
    import traceback

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import torch
        import torch.distributed as dist

        import bench
        import paper_2106_00124_b200 as ex
        from oracle import oracle as orc
        from paper_2106_00124_b200.sharded import ShardedRunner, make_local_slab
        from parity import compare, float64_oracle

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=dev)
        assert dist.get_backend() == "nccl"
        ext, box = (64, 96, 1024), (16, 16, 16)
        for route, mono in (("box-complement", "add-f32"), ("bdbsc", "add-f32"),
                            ("bdbs", "add-f32"), ("box-complement", "max-i64")):
            ops = ex.resolve_monoid(mono)
            cfg = "c4" if mono == "add-f32" else "c2"
            x = make_local_slab(lambda p0, p1: bench.make_input(cfg, dev, shape=ext, planes=(p0, p1)),
                                ext, 0, 1, box)
            runner = ShardedRunner(route, ops, ext, box, 0, 1, dev)
            got = runner(x).cpu().numpy()
            a = x.cpu().numpy()
            op = "max" if mono == "max-i64" else "add"
            # bdbs: bit-exact against the oracle in the data's own type
            want = (orc.ROUTES[route](a, box, op) if route == "bdbs"
                    else float64_oracle(route, a, box, orc, op))
            ok, ratio, rel = compare(route, got, want, a, box, orc)
            assert ok, (route, mono, ratio, rel)
        dist.destroy_process_group()
        q.put("ok")
    except Exception:  # pragma: no cover - reported to the parent
        q.put(traceback.format_exc())


def test_nccl_world1_sharded_routes():
    """the NCCL code path of ShardedRunner (world size 1 -- the
    GPU boxes of this run have one GPU) against the oracle for all routes."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(port, q))
    p.start()
    msg = q.get(timeout=600)
    p.join(timeout=60)
    assert msg == "ok", msg
