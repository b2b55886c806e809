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


def _ceilings():
    """Same-size ceilings from tools/bw_probe.cu (profiles/r2_bw_probe.jsonl): the best grid's
    average GB/s of a plain read / write / copy kernel per traffic size, L2 flushed the same
    way as kernel_report does."""
    best = {}
    try:
        for line in open(os.path.join(ROOT, "profiles", "r2_bw_probe.jsonl")):
            r = json.loads(line)
            key = (r["kind"], r["traffic_MB"])
            best[key] = max(best.get(key, 0.0), float(r["GBps_avg"]))
    except OSError:
        pass
    return best


def _ceiling_gbs(best, name):
    """Plain-kernel GB/s at this launch's traffic size (log-interpolated between probe sizes)."""
    import math
    if not best or "MB]" not in name:
        return None
    mb = float(name.split("[")[1].rstrip("MB]"))
    base = name.split("[")[0]
    kind = "read" if base in ("idem_scan", "total", "row_reduce") else \
        "write" if base == "idem_bcast" else "copy"
    pts = sorted((m, g) for (k, m), g in best.items() if k == kind)
    if not pts or mb < pts[0][0] * 0.5:
        return None
    if mb <= pts[0][0]:
        return pts[0][1]
    for (m0, g0), (m1, g1) in zip(pts, pts[1:]):
        if mb <= m1:
            t = (math.log(mb) - math.log(m0)) / (math.log(m1) - math.log(m0))
            return g0 + t * (g1 - g0)
    return pts[-1][1]


def main(path):
    ceil = _ceilings()
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
    print(f"| config | route | operator | box | step ms | G elem/s | pass (algorithmic MB) | pass ms | TB/s | of measured {PEAK / 1000:.2f} | of nominal 8 | of a plain kernel with the same traffic | dimension passes in the launch | >= 70% of measured (per dimension pass) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
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
            cg = _ceiling_gbs(ceil, name)
            print(f"{lead} {name} | {k.get('ms', 0):.3f} | {gbs / 1000:.2f} | {gbs / PEAK:.2f} | "
                  f"{gbs / NOMINAL:.2f} | {f'{gbs / cg:.2f}' if cg else '--'} | {m if m else '--'} | {mark} |")
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
