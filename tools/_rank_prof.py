import os, sys
sys.path.insert(0, "/root/repo")
import torch, bench
import paper_2106_00124_b200 as ex
from paper_2106_00124_b200 import sharded, _native
dev = torch.device("cuda", 0)
ext, dtype, box, _, _ = bench.CONFIGS["c4"]
a = bench.make_input("c4", dev)
ops = ex.Float32AddOps()
engine = sharded.CudaEngine(ops, dev)
for route in ("box-complement", "bdbs"):
    for _ in range(2):
        sharded.run_loopback(route, ops, a, box, 8, engine, concat=False)
    torch.cuda.synchronize()
    _native.profile_enable(True)
    sharded.run_loopback(route, ops, a, box, 8, engine, concat=False)
    torch.cuda.synchronize()
    recs = _native.profile_records()
    _native.profile_enable(False)
    print(route, "launches", len(recs), "sum ms", sum(r[2] for r in recs))
    # rank 3's share: records are in launch order; print the distinct (name, MB) with count and mean
    agg = {}
    for name, b, ms in recs:
        k = (name, round(b / 2**20))
        d = agg.setdefault(k, [0, 0.0]); d[0] += 1; d[1] += ms
    for k, (n, ms) in agg.items():
        print("   ", k, n, "launches, mean us", round(ms / n * 1e3, 1), "GB/s", round(k[1] * 2**20 / (ms / n * 1e-3) / 1e9) if ms else 0)
