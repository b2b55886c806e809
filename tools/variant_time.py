"""Time one route/config under several builds of the library (EXSUM_LIB ablations).

    python tools/variant_time.py --config c2 --route box-complement --op max a.so b.so ...

For each library a fresh process runs the route with per-kernel CUDA-event
profiling (L2 flushed before every call when the arrays are under 4x L2) and
prints the median step time and each kernel's median time.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r'''
import json, os, statistics, sys
sys.path.insert(0, %(root)r)
import torch
import bench
import paper_2106_00124_b200 as ex
from paper_2106_00124_b200 import _native
cfg, route, op, reps = %(cfg)r, %(route)r, %(op)r, %(reps)d
ext, dtype, box, _, _ = bench.CONFIGS[cfg]
if %(box)r: box = tuple(%(box)r)
x = bench.make_input(cfg, "cuda", shape=tuple(%(shape)r) or None)
ops = {("int64","max"): ex.IntMaxOps(), ("int64","add"): ex.IntAddOps(), ("float32","add"): ex.Float32AddOps(),
       ("float64","add"): ex.FloatAddOps()}[(dtype, op)]
fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded, "box-complement": ex.box_complement_excluded}[route]
t = ex.Tensor(ops, x)
# L2 flush by READING 512 MB (clean lines: no write-back lands in the timed call)
flush = torch.ones(64 * 2**20, dtype=torch.float64, device="cuda") if x.numel() * x.element_size() < 4 * 126e6 else None
for _ in range(3): fn(t, box)
steps, kern = [], {}
for i in range(reps):
    if flush is not None: flush.sum()
    torch.cuda.synchronize()
    _native.profile_enable(True)
    torch.cuda._sleep(400000)  # the device spins while the host enqueues the call
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); o = fn(t, box); b.record(); torch.cuda.synchronize()
    steps.append(a.elapsed_time(b))
    for name, by, ms in _native.profile_records():
        kern.setdefault(name, []).append(ms)
    _native.profile_enable(False)
    del o
plain = []
for i in range(reps):
    if flush is not None: flush.sum()
    torch.cuda._sleep(400000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); o = fn(t, box); b.record(); torch.cuda.synchronize()
    plain.append(a.elapsed_time(b)); del o
print(json.dumps({"step_ms": statistics.median(plain), "step_ms_profiled": statistics.median(steps),
                  "kernels": {k: statistics.median(v) / (len(v) / reps) * 1.0 for k, v in kern.items()}}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--route", default="box-complement")
    ap.add_argument("--op", default="max")
    ap.add_argument("--box", default="")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shape", default="", help="extents instead of the config's (same dtype)")
    ap.add_argument("libs", nargs="*")
    args = ap.parse_args()
    box = [int(v) for v in args.box.split(",")] if args.box else []
    libs = args.libs or [""]
    for lib in ["default"] + [l for l in libs if l]:
        env = dict(os.environ)
        if lib != "default":
            env["EXSUM_LIB"] = os.path.abspath(lib)
        shape = [int(v) for v in args.shape.split(",")] if args.shape else []
        code = CHILD % {"root": ROOT, "cfg": args.config, "route": args.route, "op": args.op,
                        "reps": args.reps, "box": box, "shape": shape}
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
        print(os.path.basename(lib), line, flush=True)


if __name__ == "__main__":
    main()
