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
    print(f"| config | route | operator | box | step ms | G elem/s | pass (algorithmic MB) | pass ms | TB/s | of measured {PEAK / 1000:.2f} | of nominal 8 | dimension passes in the launch | >= 70% of measured (per dimension pass) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for d in rows:
        ks = d["kernels"] or {"(launch-bound, no per-launch records)": {"ms": 0, "GBps": 0}}
        nper = _passes_per_kernel(d)
        first = True
        for name, k in ks.items():
            gbs = k.get("GBps", 0.0)
            big = "MB]" in name and float(name.split("[")[1].rstrip("MB]")) >= 100
            m = nper.get(name)
            eq = gbs * (m or 1)
            mark = ("yes" if eq >= 0.7 * PEAK else "no") if big else "n/a (small)"
            if big and m and m > 1:
                mark += f" ({eq / PEAK:.2f} per pass)"
            lead = (f"| {d['config']} | {d['route']} | {d['op']} | {'x'.join(map(str, d['box']))} | "
                    f"{d['step_ms']:.3f} | {d['Gelem_s']:.1f} |") if first else "| | | | | | |"
            print(f"{lead} {name} | {k.get('ms', 0):.3f} | {gbs / 1000:.2f} | {gbs / PEAK:.2f} | "
                  f"{gbs / NOMINAL:.2f} | {m if m else '--'} | {mark} |")
            first = False


def _passes_per_kernel(d):
    """Dimension passes each launch of a bdbs / bdbsc step carries: 1 for a
    single pass, 2 for fused_pair / outer_pair, the rest of the route's passes
    (axes with k > 1) for block_fused.  Other routes: unknown (None)."""
    if d["route"] not in ("bdbs", "bdbsc"):
        return {}
    P = sum(1 for k in d["box"] if k > 1)
    out, rest = {}, P
    launches = {name: max(1, round(v.get("ms", 0) and 1)) for name, v in d["kernels"].items()}
    for name in d["kernels"]:
        base = name.split("[")[0]
        if base in ("pass_strided", "pass_rows"):
            out[name] = None  # per-kernel rows may aggregate several single passes
        elif base in ("fused_pair", "outer_pair"):
            out[name] = 2
            rest -= 2
    for name in d["kernels"]:
        if name.split("[")[0] == "block_fused":
            singles = sum(1 for n in d["kernels"] if n.split("[")[0] in ("pass_strided", "pass_rows"))
            out[name] = None if singles else max(rest, 1)
    del launches
    return out

if __name__ == "__main__":
    main(sys.argv[1])
