"""Time BDBS on a C1-shaped array for several dtypes (tile-pair probe)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2106_00124_b200 as ex

    flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
    for name, dt, ops in (("f64", torch.float64, ex.FloatAddOps()), ("f32", torch.float32, ex.Float32AddOps()),
                          ("i64", torch.int64, ex.IntAddOps())):
        for shape in ((1024, 1024), (2048, 2048)):
            x = (torch.rand(shape, device="cuda", dtype=torch.float64) * 100).to(dt)
            t = ex.Tensor(ops, x)
            for _ in range(3):
                ex.bdbs_included(t, (32, 32))
            ts = []
            for _ in range(20):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                o = ex.bdbs_included(t, (32, 32))
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
                del o
            ts.sort()
            print(name, shape, "median %.4f ms  min %.4f" % (ts[len(ts) // 2], ts[0]), flush=True)


if __name__ == "__main__":
    main()
