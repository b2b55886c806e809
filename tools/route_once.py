"""Run one route a few times on a seeded BASELINE-shaped array -- an ncu target.

    python tools/route_once.py --config c4 --route box-complement [--box 16,16,16] [--reps 3]
    python tools/route_once.py --config c1 --shape 4096,4096 --dtype int64 --op max --route bdbs --box 4,4
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--route", default="box-complement")
    ap.add_argument("--box", default="")
    ap.add_argument("--shape", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtype", default="", help="override the config's dtype (float32/float64/int64)")
    ap.add_argument("--op", default="", help="add / max (int64 only)")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2106_00124_b200 as ex

    ext, dtype, box, _, _ = bench.CONFIGS[args.config]
    if args.box:
        box = tuple(int(v) for v in args.box.split(","))
    shape = tuple(int(v) for v in args.shape.split(",")) if args.shape else None
    x = bench.make_input(args.config, "cuda", shape=shape)
    if args.dtype:
        dtype = args.dtype
        x = x.to(getattr(torch, dtype)) if dtype != "int64" else (x * 2**20).to(torch.int64)
    ops = bench.ops_for(ex, dtype, args.route)
    if args.op:
        ops = {("int64", "max"): ex.IntMaxOps(), ("int64", "add"): ex.IntAddOps(),
               ("float32", "add"): ex.Float32AddOps(), ("float64", "add"): ex.FloatAddOps()}[(dtype, args.op)]
    fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
          "box-complement": ex.box_complement_excluded}[args.route]
    t = ex.Tensor(ops, x)
    for _ in range(args.reps):
        o = fn(t, box)
        del o
    torch.cuda.synchronize()
    print("done", args.config, args.route, box)


if __name__ == "__main__":
    main()
