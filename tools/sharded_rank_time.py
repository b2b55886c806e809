"""GPU time of one rank's share of a sharded C4 step at world sizes 2/4/8, on one GPU.

`sharded.run_loopback` runs every virtual rank's stages in turn on slices of the one C4 array
(halo sliced from the neighbour's planes, gathers as concatenations): the same stage entry
points, split axis-0 pass (interior blocks, then the last block once the halo is there), own-rows
tail and finish kernels a real rank launches -- everything but the NCCL transfers.  Total device
time / world = what one rank computes per step; against the single-GPU step / world it is the
compute-side scaling ceiling before NCCL latencies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

import torch

import bench
import paper_2106_00124_b200 as ex
from paper_2106_00124_b200 import sharded


def main():
    dev = torch.device("cuda", 0)
    ext, dtype, box, _, _ = bench.CONFIGS["c4"]
    a = bench.make_input("c4", dev)
    for route in ("box-complement", "bdbsc", "bdbs"):
        ops = ex.Float32AddOps()
        fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
              "box-complement": ex.box_complement_excluded}[route]
        t = ex.Tensor(ops, a)

        def timed(f, reps=5):
            for _ in range(2):
                o = f()
                del o
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                o = f()
                del o
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps

        single = timed(lambda: fn(t, box))
        row = {"route": route, "single_gpu_ms": round(single, 4)}
        engine = sharded.CudaEngine(ops, dev)
        for world in (2, 4, 8):
            ms = timed(lambda: sharded.run_loopback(route, ops, a, box, world, engine, concat=False))
            row[f"world{world}_rank_ms"] = round(ms / world, 4)
            row[f"world{world}_compute_scaling"] = round(single / ms, 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
