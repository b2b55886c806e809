"""Render tools/kernel_report.py JSON lines as a markdown table of passes:
achieved bandwidth (algorithmic bytes / CUDA-event time), fraction of the
measured copy peak and of the nominal 8 TB/s, against BASELINE's 70% target.

    python tools/kr_to_md.py profiles/r1_kernel_report.jsonl > profiles/r1_passes.md
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:  # the driver-written measured copy peak of this pool's B200s
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    PEAK = 6650.0  # B200_PROFILING.md fallback
NOMINAL = 8000.0


def main(path):
    rows = []
    seen = set()
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        key = (d["config"], d["route"], d["op"], tuple(d["box"]))
        if key in seen:
            continue
        seen.add(key)
        rows.append(d)
    print(f"| config | route | operator | box | step ms | G elem/s | pass (algorithmic MB) | pass ms | TB/s | of measured {PEAK / 1000:.2f} | of nominal 8 | >= 70% of measured |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        ks = d["kernels"] or {"(launch-bound, no per-launch records)": {"ms": 0, "GBps": 0}}
        first = True
        for name, k in ks.items():
            gbs = k.get("GBps", 0.0)
            big = "MB]" in name and float(name.split("[")[1].rstrip("MB]")) >= 100
            mark = ("yes" if gbs >= 0.7 * PEAK else "no") if big else "n/a (small)"
            lead = (f"| {d['config']} | {d['route']} | {d['op']} | {'x'.join(map(str, d['box']))} | "
                    f"{d['step_ms']:.3f} | {d['Gelem_s']:.1f} |") if first else "| | | | | | |"
            print(f"{lead} {name} | {k.get('ms', 0):.3f} | {gbs / 1000:.2f} | {gbs / PEAK:.2f} | "
                  f"{gbs / NOMINAL:.2f} | {mark} |")
            first = False


if __name__ == "__main__":
    main(sys.argv[1])
