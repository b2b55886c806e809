"""Run one windowed pass (exsum_windowed_pass) a few times -- an ncu target.

    python tools/one_pass.py --shape 1024,1024,1024 --axis 2 --k 16 --dtype float32 [--op add] [--reps 3]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1024,1024,1024")
    ap.add_argument("--axis", type=int, default=2)
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--op", default="add")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--route", default="")
    args = ap.parse_args()
    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200 import _native

    shape = tuple(int(v) for v in args.shape.split(","))
    tdt = {"float32": torch.float32, "float64": torch.float64, "int64": torch.int64}[args.dtype]
    x = torch.rand(shape, device="cuda", dtype=torch.float64).mul(1000).to(tdt)
    out = torch.empty_like(x)
    L = _native.load()
    stream = torch.cuda.current_stream().cuda_stream
    if args.route:
        ops = ex.resolve_monoid({"float32": "add-f32", "float64": "add-f64"}.get(args.dtype, "max-i64" if args.op == "max" else "add-i64"))
        fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
              "box-complement": ex.box_complement_excluded, "sat": ex.sat_included,
              "satc": ex.sat_excluded}[args.route]
        t = ex.Tensor(ops, x)
        for _ in range(args.reps):
            fn(t, (args.k,) * len(shape))
    else:
        for _ in range(args.reps):
            _native.check(L.exsum_windowed_pass(x.data_ptr(), out.data_ptr(), _native.DTYPE[args.dtype],
                                                _native.OP[args.op], len(shape),
                                                _native.i64_array(shape), args.axis, args.k, stream))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
