"""Time the reference's own numpy implementation (single-threaded) on samples
of the BASELINE configs -- the "reference CPU path" of BASELINE.md section 2.

Runs ONLY in the build container: it imports the unmodified reference package
read-only from /root/reference/pkg/src (which does not exist on the GPU box),
so the figure is taken on this container's host CPU, not the GPU box's, and
is reported as a labelled side figure (profiles/r2_reference_numpy.json); the
bench's reference arm times the C port (oracle/) on the GPU box itself.

    python tools/time_reference_numpy.py [--planes 16]

Each case runs the reference entry point exactly as its bench does
(bench.py:206-229: fn(Tensor(ops, arr), box)) on the leading `planes` planes
of the config's array (seeded numpy values of the config's distribution),
timed with perf_counter, and reports elements/s; float32 uses the test-side
subclass of the reference's FloatAddOps that SURVEY 8(c) prescribes.
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--planes", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_reference_numpy.json"))
    args = ap.parse_args()
    if not os.path.isdir(REF_SRC):
        print("the reference is not present here (GPU box?): nothing to time")
        return
    sys.path.insert(0, REF_SRC)
    import exsum as ref

    class AddF32(ref.FloatAddOps):
        name = "add-f32"
        dtype = np.dtype(np.float32)
        identity = np.float32(0.0)

    rng = np.random.default_rng(0)
    cases = [
        ("c4", "box-complement", AddF32(), (args.planes, 1024, 1024), (16, 16, 16),
         lambda s: rng.random(s, dtype=np.float32)),
        ("c4", "bdbsc", AddF32(), (args.planes, 1024, 1024), (16, 16, 16),
         lambda s: rng.random(s, dtype=np.float32)),
        ("c2", "box-complement", ref.IntMaxOps(), (64, 256, 256), (8, 8, 8),
         lambda s: rng.integers(-2**20, 2**20, size=s, dtype=np.int64)),
        ("c1", "bdbs", ref.FloatAddOps(), (1024, 1024), (32, 32),
         lambda s: rng.random(s, dtype=np.float64)),
    ]
    fns = {"bdbs": ref.bdbs_included, "bdbsc": ref.bdbs_excluded,
           "box-complement": ref.box_complement_excluded}
    lines = []
    for cfg, route, ops, shape, box, gen in cases:
        a = gen(shape)
        t = ref.Tensor(ops, a)
        t0 = time.perf_counter()
        fns[route](t, box)
        dt = time.perf_counter() - t0
        rec = {"config": cfg, "route": route, "operator": ops.name, "sample_extents": list(shape),
               "box": list(box), "seconds": dt, "elements_per_s": a.size / dt,
               "threads": 1, "host": _cpu_model(),
               "where": "build container (reference not available on the GPU box)",
               "numpy": np.__version__}
        print(json.dumps(rec), flush=True)
        lines.append(rec)
    with open(args.out, "w") as f:
        json.dump(lines, f, indent=1)


if __name__ == "__main__":
    main()
