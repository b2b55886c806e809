"""Step time of repeated device calls with and without CUDA-graph replay.

    EXSUM_GRAPH=0 python tools/graph_bench.py   # direct launches every call
    python tools/graph_bench.py                 # replayed graphs (default)

Profiler off (it disables replay); CUDA events around 50 back-to-back calls
with the same tensors after 5 warm-ups; one JSON line per (config, route).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [
    ("c1", (1024, 1024), "add-f64", (32, 32), "bdbs"),
    ("c2", (256, 256, 256), "max-i64", (8, 8, 8), "box-complement"),
    ("c2", (256, 256, 256), "add-i64", (8, 8, 8), "bdbsc"),
    ("c3a", (4096, 4096), "add-f32", (4, 4), "bdbs"),
    ("c3b", (256, 256, 256), "add-f32", (4, 4, 4), "bdbs"),
    ("c3c", (64,) * 4, "add-f32", (4,) * 4, "bdbs"),
    ("c3d", (28,) * 5, "add-f32", (4,) * 5, "bdbs"),
    ("c3e", (16,) * 6, "add-f32", (4,) * 6, "bdbs"),
    ("c3e", (16,) * 6, "max-i64", (4,) * 6, "bdbs"),
]


def main():
    import torch

    import paper_2106_00124_b200 as ex

    for cfg, shape, mono, box, route in CASES:
        g = torch.Generator(device="cuda").manual_seed(0)
        if mono.endswith("i64"):
            x = torch.randint(-2**20, 2**20, shape, device="cuda", dtype=torch.int64, generator=g)
        else:
            x = torch.rand(shape, device="cuda", dtype=torch.float32 if mono == "add-f32" else torch.float64,
                           generator=g)
        ops = ex.Float32AddOps() if mono == "add-f32" else ex.resolve_monoid(mono)
        fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
              "box-complement": ex.box_complement_excluded}[route]
        t = ex.Tensor(ops, x)
        out = torch.empty_like(x)
        L = ex._native.load()
        from paper_2106_00124_b200.routes import run_device
        k = ex.normalize_box(shape, box)
        dt = {torch.float32: "float32", torch.float64: "float64", torch.int64: "int64"}[x.dtype]
        op = "max" if mono.startswith("max") else "add"
        for _ in range(5):
            run_device(route, x, dt, op, shape, k, out=out)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        reps = 50
        a.record()
        for _ in range(reps):
            run_device(route, x, dt, op, shape, k, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(json.dumps({"config": cfg, "route": route, "op": mono, "box": list(box),
                          "graph": os.environ.get("EXSUM_GRAPH", "1") != "0",
                          "step_ms": round(ms, 4), "launches": L.exsum_last_launch_count()}))
        del fn, t


if __name__ == "__main__":
    main()
