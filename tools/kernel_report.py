"""Per-kernel device time and achieved HBM bandwidth for each config/route.

    python tools/kernel_report.py [--configs c1,c2,c4,...] [--reps 3]

Step time: CUDA events around each call with the profiler off (graph replay
on); arrays under 4x the 126 MB L2 get a 512 MB L2 flush (a buffer write)
before every timed call, outside its events, so no call reads its input from
the previous call's L2 lines (the 4 GiB C4 arrays are 32x L2 and need none);
per-kernel times: the library's CUDA-event profiler (exsum_profile_*), every launch
bracketed by events on its own stream; bytes are the kernel's algorithmic
(compulsory) bytes.  Prints one JSON object per (config, route).
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    "c1": ((1024, 1024), "float64", [(32, 32)], ["bdbs"]),
    "c2": ((256, 256, 256), "int64", [(8, 8, 8)], ["box-complement:max", "bdbsc", "bdbs:max"]),
    "c3a": ((4096, 4096), "float32", [(4, 4)], ["bdbs", "bdbs-i64:max"]),
    "c3b": ((256, 256, 256), "float32", [(4, 4, 4)], ["bdbs", "bdbs-i64:max"]),
    "c3c": ((64, 64, 64, 64), "float32", [(4,) * 4], ["bdbs", "bdbs-i64:max"]),
    "c3d": ((28,) * 5, "float32", [(4,) * 5], ["bdbs", "bdbs-i64:max"]),
    "c3e": ((16,) * 6, "float32", [(4,) * 6], ["bdbs", "bdbs-i64:max"]),
    "c4": ((1024, 1024, 1024), "float32", [(16, 16, 16)], ["box-complement", "bdbsc", "bdbs"]),
    "c5": ((512, 512, 512), "float64", [(2, 2, 2), (8, 8, 8), (32, 32, 32), (128, 4, 1), (1, 1, 512)],
           ["bdbs", "bdbsc"]),
    "c5bc": ((512, 512, 512), "float64", [(2, 2, 2), (8, 8, 8), (16, 16, 16)], ["box-complement"]),
    "c4bc": ((1024, 1024, 1024), "float32", [(4, 4, 4), (8, 8, 8), (16, 16, 16)], ["box-complement"]),
    # sat / satc and the mod-add monoid
    "c4sat": ((1024, 1024, 1024), "float32", [(16, 16, 16)], ["sat", "satc"]),
    "c1sat": ((1024, 1024), "float64", [(32, 32)], ["sat", "satc"]),
    "c3sat": ((256, 256, 256), "float32", [(4, 4, 4)], ["sat", "sat-i64"]),
    "c3csat": ((64, 64, 64, 64), "float32", [(4,) * 4], ["sat"]),
    "c3esat": ((16,) * 6, "float32", [(4,) * 6], ["sat"]),
    "c5sat": ((512, 512, 512), "float64", [(8, 8, 8)], ["sat", "satc"]),
    "c2corners": ((256, 256, 256), "int64", [(8, 8, 8)], ["corners:max", "box-complement:max"]),
    "c1corners": ((1024, 1024), "float64", [(32, 32)], ["corners", "box-complement"]),
    "c2mod": ((256, 256, 256), "int64", [(8, 8, 8)],
              ["bdbs:mod-add:1000003", "bdbsc:mod-add:1000003", "box-complement:mod-add:1000003",
               "sat:mod-add:1000003", "bdbs"]),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(CASES))
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200 import _native

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = torch.device("cuda:0")
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    L2_BYTES = 126 << 20

    def timed(fn, t, box, reps, flush):
        """Average device time of one call, each call bracketed by its own
        events (after an L2 flush when `flush`)."""
        total = 0.0
        for _ in range(reps):
            if flush:
                flush_buf.zero_()
            # the GPU spins while the host enqueues the call: the events time
            # the device, not the host's launch overhead (small configs)
            torch.cuda._sleep(400000)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            o = fn(t, box)
            b.record()
            torch.cuda.synchronize()
            total += a.elapsed_time(b)
            del o
        return total / reps

    for cname in args.configs.split(","):
        ext, dtype, boxes, routes = CASES[cname]
        g = torch.Generator(device=dev).manual_seed(0)
        xf = torch.rand(ext, generator=g, device=dev,
                        dtype=torch.float32 if dtype == "float32" else torch.float64) \
            if dtype != "int64" else None
        xi = None
        for box in boxes:
            for r in routes:
                route, _, op = r.partition(":")
                if route.endswith("-i64") or dtype == "int64":
                    route = route.replace("-i64", "")
                    if xi is None:
                        xi = torch.randint(-2**20, 2**20, ext, generator=g, device=dev)
                    x = xi
                    ops = (ex.IntMaxOps() if op == "max" else ex.resolve_monoid(op)
                           if op.startswith("mod-add:") else ex.IntAddOps())
                else:
                    x = xf
                    ops = ex.Float32AddOps() if dtype == "float32" else ex.FloatAddOps()
                fn = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
                      "box-complement": ex.box_complement_excluded, "sat": ex.sat_included,
                      "satc": ex.sat_excluded, "corners": ex.corners_excluded}[route]
                t = ex.Tensor(ops, x)
                for _ in range(5):  # includes the graph capture (second sighting)
                    fn(t, box)
                torch.cuda.synchronize()
                # step time with the profiler off (its per-launch events cost
                # 10-30% on the small configs, and it disables graph replay)
                flush = int(np.prod(ext)) * x.element_size() < 4 * L2_BYTES
                step_free = timed(fn, t, box, args.reps, flush)
                _native.profile_enable(True)
                step_prof = timed(fn, t, box, args.reps, flush)
                recs = _native.profile_records()
                _native.profile_enable(False)
                step_ms = step_free
                per = {}
                for name, by, ms in recs:
                    key = f"{name}[{by / 1e6:.0f}MB]"
                    d = per.setdefault(key, [0.0, 0.0, 0])
                    d[0] += ms
                    d[1] += by
                    d[2] += 1
                kern = {k: {"ms": v[0] / args.reps, "GBps": round(v[1] / v[0] / 1e6, 1),
                            "frac": round(v[1] / v[0] / 1e6 / peak, 3)} for k, v in per.items()}
                N = int(np.prod(ext))
                es = x.element_size()
                print(json.dumps({"config": cname, "route": route, "op": ops.name, "box": box,
                                  "step_ms": round(step_ms, 4),
                                  "step_ms_profiled": round(step_prof, 4),
                                  "l2_flush": flush,
                                  "Gelem_s": round(N / step_ms / 1e6, 2),
                                  "compulsory_frac": round(2 * N * es / step_ms / 1e6 / peak, 3),
                                  "kernels": kern}), flush=True)
                del t
        del xf, xi
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
