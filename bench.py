"""Benchmark: box sums on B200 (the driver's contract).

Workload (N=1 headline): BASELINE config 4 -- float32 1024x1024x1024 (4 GiB),
values uniform [0,1), box (16,16,16), strong excluded sum via
box-complement (the route the config names first; BDBSC is reported beside
it under "routes").  A step is one box_complement_excluded call over the whole
array with the input already resident in HBM.  The input (4 GiB) is 32x the
126 MB L2, so no L2 flush is needed between steps.  (The smaller configs,
--config c1 / c2: a 512 MB buffer is written before every timed step, outside
the step's events.)  `value` comes from K timed steps of the product path with
the library's per-launch profiler off; a second set of K steps with the
profiler on gives the per-kernel figures (`kernels`, `roofline`,
`profiled_ms_per_step`).

e2e: the same workload through the host-buffer C ABI from pinned memory, every
step copying its 4 GiB input in and its 4 GiB result out: over the K steps
exsum_route_host_batch overlaps the H2D of step i+1 with the compute of step i
and the D2H of step i-1 (full-duplex PCIe); "single_call_ms" is one isolated
call (H2D -> compute -> D2H).

Multi-GPU (torchrun, one process per GPU): the array is sharded along axis 0
(strong scaling of the fixed 1024^3 array); every rank runs the sharded
route (halo + carry exchange over NCCL, paper_2106_00124_b200/sharded.py) on
its slab and the step time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--route box-complement|bdbsc|bdbs]
    python bench.py --impl reference ...   # the CPU reference arm (oracle port)

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (extents, dtype, box, value distribution, description)
    "c4": ((1024, 1024, 1024), "float32", (16, 16, 16), "uniform01",
           "C4 3-D FMM-like excluded sum, float32 1024^3 uniform[0,1), box 16^3"),
    "c2": ((256, 256, 256), "int64", (8, 8, 8), "int20",
           "C2 3-D excluded sums, int64 256^3 uniform[-2^20,2^20), box 8^3"),
    "c1": ((1024, 1024), "float64", (32, 32), "uniform01",
           "C1 2-D included sum, float64 1024^2 uniform[0,1), box 32^2"),
    # C5 (box/aspect sweep) -- a measurement target for tools/, not a bench line
    "c5": ((512, 512, 512), "float64", (8, 8, 8), "normal",
           "C5 3-D box sweep, float64 512^3 standard normal, box 8^3"),
}
_JSON_OUT = sys.stdout
METRIC = "box-sum elements/s"
UNIT = "elements/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []  # (wall time, csv line)
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        """The timed region [t0, t1] (wall clock)."""
        self.window = (t0, t1)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        scope = "timed region"
        if self.window is not None:
            t0, t1 = self.window
            inside = [ln for t, ln in lines if t0 <= t <= t1]
            if len(inside) < 3:  # a short region: widen to the loaded window around it
                inside = [ln for t, ln in lines if t0 - 1.0 <= t <= t1 + 0.2]
                scope = "timed region +-1 s (loaded: warm-up and timed steps)"
            lines = inside
        else:
            lines = [ln for _, ln in lines]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms), "scope": scope}


def make_input(cfg, device, seed=0, shape=None, planes=None):
    """The workload's seeded synthetic array, or planes [p0, p1) of it.

    Every plane (index along axis 0) has its own Philox stream, seeded from
    (seed, plane), so any slab of the global array -- a rank's own planes plus
    its halo -- is generated exactly as the single-GPU array holds it: an N>1
    run computes on slices of the one array the N=1 run sees.  `shape`
    replaces the extents (its planes seeded the same way)."""
    import torch

    ext, dtype, box, dist, _ = CONFIGS[cfg]
    shape = tuple(shape or ext)
    p0, p1 = planes if planes is not None else (0, shape[0])
    tdt = {"float32": torch.float32, "float64": torch.float64, "int64": torch.int64}[dtype]
    out = torch.empty((p1 - p0,) + shape[1:], dtype=tdt, device=device)
    g = torch.Generator(device=device)
    for p in range(p0, p1):
        g.manual_seed((seed << 32) + p)
        if dist == "uniform01":
            torch.rand(shape[1:], generator=g, device=device, dtype=tdt, out=out[p - p0])
        elif dist == "normal":
            torch.randn(shape[1:], generator=g, device=device, dtype=tdt, out=out[p - p0])
        else:
            torch.randint(-2**20, 2**20, shape[1:], generator=g, device=device, dtype=tdt,
                          out=out[p - p0])
    return out


def bench_config(cfg, route, world, sharded_path):
    """The `config` object of the JSON line -- identical in both arms."""
    ext, dtype, box, dist, desc = CONFIGS[cfg]
    es = 4 if dtype == "float32" else 8
    N = int(np.prod(ext))
    return {"workload": cfg, "description": desc, "extents": list(ext), "box": list(box),
            "route": route, "operator": _monoid_name(dtype, route),
            "parallelism": f"axis0-shards{world}" if sharded_path else "single-gpu",
            "l2": "input 4 GiB >> 126 MB L2; no flush needed" if not _needs_flush(N * es)
            else "input under 4x the 126 MB L2: a 512 MB buffer is written between timed steps "
                 "(L2 flush), outside each step's events",
            "seed": 0}


def _needs_flush(nbytes):
    """Arrays under 4x the 126 MB L2 get an L2 flush between timed steps."""
    return nbytes < 4 * 126e6


def _monoid_name(dtype, route):
    if dtype == "float32":
        return "add-f32"
    if dtype == "float64":
        return "add-f64"
    return "max-i64" if route == "box-complement" else "add-i64"


def ops_for(ex, dtype, route):
    if dtype == "float32":
        return ex.Float32AddOps()
    if dtype == "float64":
        return ex.FloatAddOps()
    return ex.IntMaxOps() if route == "box-complement" else ex.IntAddOps()


def cpu_sample(cfg, route, nthreads, planes=64, reps=1):
    """Time the CPU oracle port (oracle/, the reference algorithm restated in C
    with OpenMP over independent lines) on a bounded sample of the workload:
    the first `planes` planes along axis 0 (same trailing shape, same value
    distribution, same box).  Returns elements/s."""
    from oracle import oracle as orc

    ext, dtype, box, dist, _ = CONFIGS[cfg]
    shape = (min(planes, ext[0]),) + tuple(ext[1:])
    rng = np.random.default_rng(0)
    if dist == "uniform01":
        a = rng.random(shape, dtype=np.float32 if dtype == "float32" else np.float64)
    else:
        a = rng.integers(-2**20, 2**20, size=shape, dtype=np.int64)
    op = "max" if (dtype == "int64" and route == "box-complement") else "add"
    fn = orc.ROUTES[route]
    best = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn(a, box, op, nthreads)
        best.append(time.perf_counter() - t0)
    dt = statistics.median(best)
    return a.size / dt, shape, dt


def _mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm on the host cores.

    The reference is pure Python + numpy (single-threaded); its
    algorithm restated in C with the reference's exact association
    (oracle/exsum_oracle.c, OpenMP over independent lines and column tiles,
    bit-identical for any thread count) runs here on every host thread.  A
    step is the WHOLE workload array -- the same extents, box, route, value
    distribution and seed as the GPU arm (same `config`); only if the host
    lacks the memory for it does the step fall back to a leading-planes
    sample, and `cpu_baseline.sample` says so.  Under torchrun only rank 0
    runs."""
    if rank != 0:
        return
    cfg = args.config
    nthreads = os.cpu_count() or 1
    ext, dtype, box, _, desc = CONFIGS[cfg]
    from oracle import oracle as orc

    es = 4 if dtype == "float32" else 8
    N = int(np.prod(ext))
    # the oracle's box-complement holds 4 N-sized scratch arrays + out + in
    need = 7 * N * es + (1 << 30)
    planes = ext[0] if _mem_available() >= need else max(1, args.cpu_planes)
    shape = (planes,) + tuple(ext[1:])
    rng = np.random.default_rng(0)
    if dtype == "int64":
        a = rng.integers(-2**20, 2**20, size=shape, dtype=np.int64)
    else:
        a = rng.random(shape, dtype=np.float32 if dtype == "float32" else np.float64)
    op = "max" if (dtype == "int64" and args.route == "box-complement") else "add"
    fn = orc.ROUTES[args.route]
    for _ in range(args.warmup):
        fn(a, box, op, nthreads)
    secs = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn(a, box, op, nthreads)
        secs.append(time.perf_counter() - t0)
    total = sum(secs)
    value = a.size * args.steps / total
    sample = (f"the whole {'x'.join(map(str, shape))} array every step" if planes == ext[0] else
              f"the first {planes} planes ({'x'.join(map(str, shape))}) every step: the host "
              f"lacks memory for the whole array")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": _dt(dtype),
        "data": "synthetic",
        "config": bench_config(cfg, args.route, world, world > 1 or args.sharded),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "cpu_model": _cpu_model(), "cpu_count": os.cpu_count(),
                         "sample": f"{args.route}: {sample}; oracle/exsum_oracle.c (the "
                                   f"reference algorithm, its association) on {nthreads} "
                                   f"OpenMP threads; values numpy default_rng(0)",
                         "whole_array": planes == ext[0]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=_JSON_OUT, flush=True)


def _cpu_model():
    """The host CPU's model string (report it beside the core count)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _dt(dtype):
    return {"float32": "f32", "float64": "f64", "int64": "int64"}[dtype]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--route", default="box-complement", choices=["box-complement", "bdbsc", "bdbs"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-planes", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", action="store_true",
                    help="after timing, compare this rank's output planes with the single-GPU "
                         "route on the whole global array (on this rank's GPU) and report it")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded, NCCL) path even at world size 1 "
                         "(run under torchrun; exercises the N>1 code on one GPU)")
    args = ap.parse_args()

    if args.sharded and "RANK" not in os.environ:
        # --sharded without torchrun: a world of one rank on this host
        os.environ.update({"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "1",
                           "MASTER_ADDR": "127.0.0.1",
                           "MASTER_PORT": os.environ.get("MASTER_PORT", "29531")})
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # stdout carries the ONE JSON line and nothing else: libraries that write to
    # fd 1 (NCCL prints its version there when NCCL_DEBUG is set on the box) go
    # to stderr from here on; the line is printed to the saved descriptor
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch

    import paper_2106_00124_b200 as ex
    from paper_2106_00124_b200 import _native

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    sharded_path = world > 1 or args.sharded
    if sharded_path:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    ext, dtype, box, _, desc = CONFIGS[args.config]
    N = int(np.prod(ext))
    es = 4 if dtype == "float32" else 8
    ops = ops_for(ex, dtype, args.route)
    fn = {"box-complement": ex.box_complement_excluded, "bdbsc": ex.bdbs_excluded,
          "bdbs": ex.bdbs_included}[args.route]

    if sharded_path:
        from paper_2106_00124_b200 import sharded

        x = sharded.make_local_slab(lambda p0, p1: make_input(args.config, dev, planes=(p0, p1)),
                                    ext, rank, world, box)
        runner = sharded.ShardedRunner(args.route, ops, ext, box, rank, world, dev)
        step = lambda: runner(x)  # noqa: E731
    else:
        x = make_input(args.config, dev)
        t = ex.Tensor(ops, x)
        step = lambda: fn(t, box)  # noqa: E731

    stream = torch.cuda.current_stream(dev)
    clocks = ClockSampler(local).__enter__()
    time.sleep(0.5)  # let nvidia-smi start sampling
    # allocated before the warm-up: the graph cache keys on the output pointer
    # the allocator hands back, which a later 512 MB allocation could move
    flush = (torch.empty(512 * 2**20, dtype=torch.uint8, device=dev)
             if _needs_flush(N * es // (world if sharded_path else 1)) else None)
    for _ in range(args.warmup):
        if flush is not None:
            flush.fill_(0)
        out = step()
        del out
    torch.cuda.synchronize(dev)

    # -- timed region: K steps, device events on the launching stream --------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    def timed_steps():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        # keep the GPU busy while the host enqueues the K steps (~0.2 ms of spin per
        # step, before the first start event): the events then time the device's
        # back-to-back execution of the steps, not the host's enqueue rate -- which
        # bounds a small config (C1: ~16 us of Python per call), and which e2e keeps
        torch.cuda._sleep(int(args.steps * 2e-4 * 1.965e9))
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i & 0xFF)  # before the start event: not in the step's time
            starts[i].record(stream)
            out = step()
            ends[i].record(stream)
            del out
        torch.cuda.synchronize(dev)
        return [a.elapsed_time(b) for a, b in zip(starts, ends)]

    # Two sets of K timed steps.  The first runs the product path as a caller
    # sees it (profiler off, so repeated calls replay the captured CUDA graph):
    # `value` / `ms_per_step` come from it.  The second has the library's
    # per-launch CUDA events on (they cost ~17 us of a 2.7 ms C4 step and a
    # quarter of a 60 us C2 step, and switch graph replay off): the `kernels`
    # and `roofline` figures and `profiled_ms_per_step` come from that one.
    # (the W warm-up steps above are the first sighting and the graph capture)
    t_begin = time.time()
    unprofiled_ms = timed_steps()
    _native.profile_enable(True)
    launches0 = _native.total_launch_count()
    profiled_ms = timed_steps()
    launches = _native.total_launch_count() - launches0
    clocks.mark(t_begin, time.time())
    time.sleep(0.1)
    clocks.__exit__(None, None, None)
    if dist is not None:
        dist.barrier()
    step_ms = unprofiled_ms
    prof = _native.profile_records()
    _native.profile_enable(False)
    total_ms = sum(step_ms)
    if dist is not None:
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = N * args.steps / (total_ms / 1e3)

    # -- roofline of the dominant kernel (per-launch events inside the region) --
    peak, peak_kind = _peaks()
    per = {}
    for name, b, ms in prof:
        key = f"{name}[{b / 2**20:.0f}MiB]"
        d = per.setdefault(key, {"ms": 0.0, "bytes": 0.0, "launches": 0})
        d["ms"] += ms
        d["bytes"] += b
        d["launches"] += 1
    dom = max(per, key=lambda k: per[k]["ms"]) if per else None
    kernels = {}
    for name, d in per.items():
        gbs = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
        kernels[name] = {"launches": d["launches"], "avg_ms": d["ms"] / d["launches"],
                         "bytes_per_launch": d["bytes"] / d["launches"], "GBps": gbs,
                         "share_of_step": d["ms"] / sum(profiled_ms) if sum(profiled_ms) else None}
    roofline = None
    if dom is not None:
        d = per[dom]
        ach = d["bytes"] / (d["ms"] / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "peak_source": peak_kind, "traffic": _ncu_traffic(dom)}
    step_bytes = sum(d["bytes"] for d in per.values()) / max(args.steps, 1)
    e2e_frac = 2 * N * es / (ms_per_step / 1e3) / 1e9 / peak

    # -- other routes on the same array, for context (not the headline) -------
    routes = {}
    if not sharded_path:
        for rname, rfn in (("bdbsc", ex.bdbs_excluded), ("bdbs", ex.bdbs_included),
                           ("box-complement", ex.box_complement_excluded)):
            if rname == args.route or (rname == "bdbsc" and not ops.has_inverse):
                continue
            rt = ex.Tensor(ops, x)
            for _ in range(2):
                rfn(rt, box)
            torch.cuda.synchronize(dev)
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            reps = 3
            for _ in range(reps):
                o = rfn(rt, box)
                del o
            b_ev.record(stream)
            torch.cuda.synchronize(dev)
            ms = a_ev.elapsed_time(b_ev) / reps
            routes[rname] = {"ms_per_step": ms, "elements_per_s": N / (ms / 1e3)}

    # -- end to end through the public API with host buffers ------------------
    e2e = None
    if not args.no_e2e and not sharded_path:
        host_in = torch.empty(ext, dtype=x.dtype, pin_memory=True)
        host_in.copy_(x)
        host_out = torch.empty_like(host_in, pin_memory=True)
        a_np, o_np = host_in.numpy(), host_out.numpy()
        from paper_2106_00124_b200.routes import run_host

        k = ex.normalize_box(ext, box)
        dname = {"float32": "float32", "float64": "float64", "int64": "int64"}[dtype]
        run_host(args.route, a_np, dname, ops.op, ext, k, out=o_np)  # warm-up (allocates the cache)
        # one call at a time (latency): H2D, compute, D2H in sequence
        single = []
        for _ in range(2):
            t0 = time.perf_counter()
            r = run_host(args.route, a_np, dname, ops.op, ext, k, out=o_np)
            single.append(time.perf_counter() - t0)
        del r
        _native.load().exsum_release_cache()
        # throughput: K arrays through exsum_route_host_batch -- every step still
        # copies its whole input in and its whole result out (pinned), but the
        # H2D of step i+1 runs while the D2H of step i drains (full-duplex PCIe)
        from paper_2106_00124_b200.routes import run_host_batch

        e_steps = max(2, min(args.steps, 12))
        run_host_batch(args.route, [a_np] * 2, dname, ops.op, ext, k, outs=[o_np] * 2)  # warm-up
        t0 = time.perf_counter()
        run_host_batch(args.route, [a_np] * e_steps, dname, ops.op, ext, k, outs=[o_np] * e_steps)
        sec = (time.perf_counter() - t0) / e_steps
        _native.load().exsum_release_cache()
        e2e = {"value": N / sec, "unit": UNIT,
               "h2d_bytes_per_step": N * es, "d2h_bytes_per_step": N * es,
               "ms_per_step": sec * 1e3, "steps": e_steps,
               "path": "exsum_route_host_batch over the steps (pinned host in/out; H2D of step "
                       "i+1 overlapped with compute of i and D2H of i-1)",
               "single_call_ms": statistics.median(single) * 1e3,
               "single_call_value": N / statistics.median(single)}

    if not args.no_e2e and sharded_path:
        # each rank: its own planes host->device, the sharded step (halo and
        # reductions over NCCL), its output planes device->host -- pipelined
        # over the steps like exsum_route_host_batch (two device slabs; the
        # H2D of step i+1 and the D2H of step i-1 overlap step i); max over ranks
        n_own = runner.n_own
        host_in = torch.empty((n_own,) + tuple(ext[1:]), dtype=x.dtype, pin_memory=True)
        host_in.copy_(x[:n_own])
        host_out = torch.empty_like(host_in, pin_memory=True)
        slabs = [x, torch.empty_like(x)]
        s_in, s_run, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_run = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def e2e_run(steps):
            for i in range(steps):
                j = i % 2
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(ev_run[j])
                    slabs[j][:n_own].copy_(host_in, non_blocking=True)
                    ev_in[j].record(s_in)
                with torch.cuda.stream(s_run):
                    s_run.wait_event(ev_in[j])
                    if i >= 2:
                        s_run.wait_event(ev_out[j])
                    y = runner(slabs[j])
                    ev_run[j].record(s_run)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_run[j])
                    if y is not None and n_own > 0:
                        host_out.copy_(y, non_blocking=True)
                        y.record_stream(s_out)
                    ev_out[j].record(s_out)
            torch.cuda.synchronize(dev)

        single = []
        e2e_run(2)  # warm-up
        for _ in range(2):
            dist.barrier()
            t0 = time.perf_counter()
            e2e_run(1)
            single.append(time.perf_counter() - t0)
        e_steps = max(2, min(args.steps, 12))
        dist.barrier()
        t0 = time.perf_counter()
        e2e_run(e_steps)
        sec = (time.perf_counter() - t0) / e_steps
        tt = torch.tensor([sec, statistics.median(single)], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sec, sec1 = float(tt[0].item()), float(tt[1].item())
        e2e = {"value": N / sec, "unit": UNIT, "h2d_bytes_per_step": N * es,
               "d2h_bytes_per_step": N * es, "ms_per_step": sec * 1e3, "steps": e_steps,
               "path": "per rank: own planes H2D (pinned) + ShardedRunner + own output D2H, "
                       "pipelined over the steps on two slabs; max over ranks; bytes summed "
                       "over ranks",
               "single_call_ms": sec1 * 1e3, "single_call_value": N / sec1}

    check = None
    if args.check:
        # the sharded ranks hold slices of one seeded global array (make_input
        # seeds every plane): their planes must equal the single-GPU route's
        y = step()
        full = make_input(args.config, dev)
        ref = fn(ex.Tensor(ops, full), box).data
        if sharded_path:
            ref = ref[runner.start:runner.end]
        diff = (y.double() - ref.double()).abs().max().item() if y is not None and y.numel() else 0.0
        mag = ref.double().abs().max().item() if ref.numel() else 0.0
        stats = torch.tensor([diff, mag], device=dev, dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(stats, op=dist.ReduceOp.MAX)
        check = {"against": "single-GPU route on the whole global array, each rank its planes",
                 "max_abs_diff": stats[0].item(), "max_abs_value": stats[1].item(),
                 "bit_exact": stats[0].item() == 0.0}
        del y, full, ref

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        nthreads = os.cpu_count() or 1
        v, shape, dt = cpu_sample(args.config, args.route, nthreads, planes=args.cpu_planes)
        cpu = {"value": v, "unit": UNIT, "cores": nthreads, "kind": "port",
               "cpu_model": _cpu_model(), "cpu_count": os.cpu_count(),
               "sample": f"{args.route} on the first {shape[0]} planes ({'x'.join(map(str, shape))}) "
                         f"of the workload, oracle/exsum_oracle.c, {nthreads} OpenMP threads, "
                         f"{dt:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,  # the 1024^3 array is fixed as N grows
            "dtype": _dt(dtype), "data": "synthetic",
            "config": bench_config(args.config, args.route, world, sharded_path),
            "roofline": roofline,
            "hbm_GBps_step": step_bytes / (ms_per_step / 1e3) / 1e9,
            "e2e_fraction_of_peak": e2e_frac,
            "kernels": kernels,
            "routes": routes,
            "gpu_launches": launches,
            "profiled_ms_per_step": sum(profiled_ms) / args.steps,
            "timed_regions": "value / ms_per_step: K steps, profiler off (repeated calls replay "
                             "the captured CUDA graph, the product path); kernels / roofline: a "
                             "second set of K steps with per-launch CUDA events",
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if check is not None:
            line["check"] = check
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from
    the committed ncu --set full capture (profiles/ncu_traffic.json), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rec = json.load(f).get(kernel)
        return rec["dram_bytes_per_launch"] if rec else None
    except Exception:
        return None


if __name__ == "__main__":
    main()
