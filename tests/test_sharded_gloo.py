"""Multi-GPU orchestration on CPU: world_size 2 with the gloo backend.

Each rank holds its k0-aligned slab (+ halo room), runs the real sharded
orchestration (paper_2106_00124_b200/sharded.py: halo exchange over
isend/irecv, all-gathers, rank-order totals, tail slicing) with the oracle in
place of the CUDA stages, and checks its output planes against the unsharded
oracle on the full array.
"""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [
    # (extents, box, route, op, dtype)
    ((37, 6, 5), (4, 3, 2), "bdbs", "add", np.int64),
    ((37, 6, 5), (4, 3, 2), "bdbsc", "add", np.int64),
    ((37, 6, 5), (4, 3, 2), "box-complement", "add", np.int64),
    ((37, 6, 5), (4, 3, 2), "box-complement", "max", np.int64),
    ((16, 9), (5, 3), "box-complement", "max", np.int64),
    ((16, 9), (5, 3), "bdbs", "max", np.int64),
    ((5, 3, 4), (8, 2, 2), "box-complement", "add", np.int64),   # one rank empty
    ((5, 3, 4), (8, 2, 2), "box-complement", "max", np.int64),   # marginal form, one rank empty
    ((20, 4, 6), (3, 2, 3), "bdbs", "add", np.float64),          # bit-exact float BDBS
    ((20, 4, 6), (3, 2, 3), "bdbsc", "add", np.float64),
    ((20, 4, 6), (3, 2, 3), "box-complement", "add", np.float32),
]


def _worker(rank, world, init_file, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle import oracle as orc
    from paper_2106_00124_b200 import resolve_monoid
    from paper_2106_00124_b200.sharded import DistComm, ShardedRunner, make_local_slab
    from parity import float_tolerance
    from shard_engines import OracleEngine

    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    try:
        for ci, (ext, box, route, op, dt) in enumerate(CASES):
            rng = np.random.default_rng(ci)
            if np.dtype(dt).kind == "i":
                a = rng.integers(-2**20, 2**20, size=ext).astype(dt)
            else:
                a = rng.standard_normal(ext).astype(dt)
            name = {("add", np.int64): "add-i64", ("max", np.int64): "max-i64",
                    ("add", np.float64): "add-f64", ("add", np.float32): "add-f32"}[(op, dt)]
            ops = resolve_monoid(name)
            engine = OracleEngine(op, np.dtype(dt).name)
            runner = ShardedRunner(route, ops, ext, box, rank, world, torch.device("cpu"),
                                   comm=DistComm(rank, world), engine=engine)
            x = make_local_slab(lambda p0, p1: torch.from_numpy(a[p0:p1].copy()), ext, rank,
                                world, box)
            out = runner(x)
            if route == "box-complement" or (route == "bdbsc" and np.dtype(dt).kind == "f"):
                src = a.astype(np.float64) if np.dtype(dt).kind == "f" else a
                want = orc.ROUTES[route](src, box, op)[runner.start:runner.end]
            else:
                want = orc.ROUTES[route](a, box, op)[runner.start:runner.end]
            if out is None:
                assert runner.n_own == 0
                continue
            got = out.numpy()
            if np.dtype(dt).kind == "f" and route != "bdbs":
                # the exactness contract of tests/parity.py on this rank's planes
                k = tuple(min(b, n) for b, n in zip(box, ext))
                tol = float_tolerance(route, a, k, orc)[runner.start:runner.end]
                assert np.all(np.abs(got.astype(np.float64) - want) <= tol), (ci, route)
            else:
                assert np.array_equal(got, want.astype(got.dtype)), (ci, route, rank)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as td:
        init_file = os.path.join(td, "init")
        procs = [ctx.Process(target=_worker, args=(r, world, init_file, q)) for r in range(world)]
        for p in procs:
            p.start()
        results = [q.get(timeout=240) for _ in range(world)]
        for p in procs:
            p.join(timeout=60)
    for rank, msg in results:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_slab_plan():
    from paper_2106_00124_b200.sharded import SlabPlan

    p = SlabPlan(1024, 16, 8)
    assert [p.bounds(r) for r in range(8)] == [(128 * r, 128 * (r + 1)) for r in range(8)]
    assert [p.halo(r) for r in range(8)] == [15] * 7 + [0]
    p = SlabPlan(37, 4, 3)
    assert [p.bounds(r) for r in range(3)] == [(0, 16), (16, 28), (28, 37)]
    assert all(b[0] % 4 == 0 for b in (p.bounds(r) for r in range(3)))
    p = SlabPlan(5, 5, 2)
    assert p.bounds(1) == (5, 5) and p.halo(0) == 0


def test_grouped_halo_only_when_every_rank_posts():
    """batch_isend_irecv needs every rank in the group: it is used only when
    every rank owns planes and every rank but the last receives a halo."""
    from paper_2106_00124_b200.sharded import DistComm, SlabPlan

    c = DistComm.__new__(DistComm)
    c.grouped = True
    for world, plan, want in ((8, SlabPlan(1024, 16, 8), True), (2, SlabPlan(37, 4, 2), True),
                              (2, SlabPlan(5, 5, 2), False),     # rank 1 owns nothing
                              (3, SlabPlan(37, 1, 3), False),    # k0 = 1: no halo at all
                              (1, SlabPlan(64, 16, 1), False)):
        c.world = world
        assert c._all_ranks_exchange(plan) is want, (world, plan)
