import json, sys
for path in sys.argv[1:]:
    for l in open(path):
        try:
            d = json.loads(l)
        except Exception:
            continue
        ks = " ".join(f"{k}:{v['ms']:.3f}ms/{v['GBps']:.0f}" for k, v in d["kernels"].items() if v["ms"] > 0.02)
        print(d["config"], d["route"], d["op"], d["box"], d["step_ms"], d["Gelem_s"], ks)
