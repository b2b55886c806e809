"""L2-pipelined schedule (csrc/l2pipe.cu, EXSUM_L2PIPE=1) against the default
two-kernel schedule: bit-equality for bdbs, closeness for box-complement, and
CUDA-event times of both.

    python tools/l2pipe_check.py [--shapes 64x256,128x1024,1024x1024] [--reps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="64x256,128x1024,1024x1024")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2106_00124_b200 as ex

    ex._native.load()
    ops = ex.Float32AddOps()
    for sh in args.shapes.split(","):
        n0, n1 = (int(v) for v in sh.split("x"))
        x = torch.rand((n0, n1, 1024), device="cuda", dtype=torch.float32, generator=torch.Generator("cuda").manual_seed(0))
        for route, fn in (("bdbs", ex.bdbs_included), ("box-complement", ex.box_complement_excluded)):
            res = {}
            for mode in ("0", "1"):
                os.environ["EXSUM_L2PIPE"] = mode
                ex.routes._PLAN_CACHE.clear()  # the workspace size depends on the schedule
                out = fn(ex.Tensor(ops, x), (16, 16, 16)).data
                torch.cuda.synchronize()
                ts = []
                for _ in range(args.reps):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn(ex.Tensor(ops, x), (16, 16, 16))
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                res[mode] = (out, min(ts), ex._native.last_launch_count())
            o0, o1 = res["0"][0], res["1"][0]
            if route == "bdbs":
                same = bool(torch.equal(o0.view(torch.int32), o1.view(torch.int32)))
                diff = 0.0
            else:
                diff = float(((o0.double() - o1.double()).abs() / o0.double().abs().clamp_min(1.0)).max())
                same = diff < 1e-5
            print(f"{sh}x1024 {route}: two-kernel {res['0'][1]:.3f} ms ({res['0'][2]} launches), "
                  f"l2pipe {res['1'][1]:.3f} ms ({res['1'][2]} launches), match={same} rel={diff:.2e}",
                  flush=True)
    os.environ["EXSUM_L2PIPE"] = "0"


if __name__ == "__main__":
    main()
