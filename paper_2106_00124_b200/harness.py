"""Benchmark harness over the B200 routes -- the caller of the hot path
(SURVEY 8(f) row 1), mirroring the reference's ``exsum.bench`` (bench.py:1-263).

Same API and CSV schema as the reference: ``run_benchmark``, ``run_sweep``,
``BenchResult.csv_row`` and ``CSV_HEADER``
(``algo,d,N,K,time_ns_per_elem,oplus_per_elem,peak_bytes_per_elem,verified``),
so scripts written against ``exsum run`` / ``exsum sweep`` read the same
columns.  The differences are the ones a GPU implies:

* ``time_ns_per_elem`` is the median wall time of ``trials`` calls of the
  registry entry (``AlgorithmInfo.run``, bench.py:54-57).  With
  ``device="host"`` (default) the tensor is numpy, so every call includes the
  host->device and device->host copies (the plug-in's real cost); with
  ``device="cuda"`` the tensor is resident in HBM and each call is bracketed by
  ``torch.cuda.synchronize()``.
* ``oplus_per_elem`` is ``NA``: the kernels apply the operator in registers
  and nothing counts the applications (the reference's ``InstrumentedMonoid``
  has no GPU meaning).
* ``peak_bytes_per_elem`` is the device memory the call needs -- input,
  output and the workspace ``exsum_route_workspace_bytes`` reports -- per
  input element (the analogue of the reference's AllocationTracker peak).
* ``verify`` checks the result against a brute-force fold over every box (or
  complement) with the monoid's scalar ``combine`` -- the reference's
  ``verify_against_oracle`` (bench.py:116-131, oracle.py:37-71), capped at
  ``VERIFY_ELEMENT_CAP`` elements like the reference.  It only checks; the
  returned result is always the GPU's.
"""

from __future__ import annotations

import math
import statistics
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigurationError, UsageError
from .monoid import device_operator, modulus_of, resolve_monoid, unwrap
from .routes import ALGORITHMS, check_algorithm_config, resolve_algorithm
from .tensor import Tensor, is_torch, normalize_box, validate_extents

CSV_HEADER = "algo,d,N,K,time_ns_per_elem,oplus_per_elem,peak_bytes_per_elem,verified"

VERIFY_ELEMENT_CAP = 4096
FLOAT_RTOL = 1e-9  # bench.py:42 (float64); float32 results use 64 float32 ulps instead
_F32_RTOL = 64 * float(np.finfo(np.float32).eps)
_DT_NAME = {np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
            np.dtype(np.int64): "int64"}


def generate_input(ops, extents, seed: int) -> Tensor:
    """Deterministic input matched to the monoid's domain (bench.py:103-114):
    floats uniform in [0, 1), integers in [0, 100) (reduced mod m for mod-add)."""
    ext = validate_extents(extents)
    rng = np.random.default_rng(seed)
    base = unwrap(ops)
    if np.dtype(base.dtype).kind == "f":
        arr = rng.random(ext)
    else:
        arr = rng.integers(0, 100, size=ext, dtype=np.int64)
        m = modulus_of(base)
        if m:
            arr %= m
    return Tensor(ops, np.ascontiguousarray(arr, dtype=base.dtype))


# -- verification (the reference's brute-force oracle, oracle.py:37-71) --------


def _fold(sel: np.ndarray, ops):
    """Row-major left fold of ``sel`` with ``ops.combine`` (identity if empty),
    vectorised per monoid with the same result as the scalar loop."""
    if sel.size == 0:
        return ops.identity
    if sel.size == 1:
        return sel[0].item()  # no combine: the raw value (oracle.py:46-52)
    name = getattr(ops, "name", "")
    if name == "max-i64":
        return int(sel.max())
    if name == "add-i64":
        return int(np.sum(sel, dtype=np.int64))  # wraps like IntAddOps.combine
    if name.startswith("mod-add:"):
        m = modulus_of(ops)
        return int(np.sum(np.mod(sel, m), dtype=np.int64)) % m
    if sel.dtype.kind == "f":
        return np.add.accumulate(sel)[-1].item()  # sequential, in the data type
    acc = sel[0].item()
    for v in sel[1:]:
        acc = ops.combine(acc, v.item())
    return acc


def _brute(kind: str, data: np.ndarray, box, ops):
    """Fold every clipped box (kind "included") or its complement ("excluded")
    in row-major order -- the reference's oracle_included / oracle_excluded."""
    ext = data.shape
    flat = data.reshape(-1)
    coords = np.indices(ext).reshape(len(ext), -1)
    out = []
    for f in range(flat.size):
        x = coords[:, f]
        inside = np.ones(flat.size, dtype=bool)
        for j, (xj, kj) in enumerate(zip(x, box)):
            inside &= (coords[j] >= xj) & (coords[j] < xj + kj)
        out.append(_fold(flat[inside if kind == "included" else ~inside], ops))
    return out


def _matches(result: np.ndarray, expected, dtype) -> bool:
    got = np.asarray(result).reshape(-1)
    if np.dtype(dtype).kind == "f":
        want = np.asarray(expected, dtype=np.float64)
        rtol = FLOAT_RTOL if np.dtype(dtype) == np.float64 else _F32_RTOL
        g = got.astype(np.float64)
        tol = rtol * np.maximum(1.0, np.maximum(np.abs(g), np.abs(want)))
        return bool(np.all(np.abs(g - want) <= tol))
    return bool(np.array_equal(got, np.asarray(expected, dtype=np.int64)))


def verify_against_oracle(info, t: Tensor, box, result: Tensor) -> bool:
    """bench.py:116-131: compare with the brute-force fold (small inputs only)."""
    base = unwrap(t.ops)
    data = t.data.cpu().numpy() if is_torch(t.data) else np.asarray(t.data)
    res = result.data.cpu().numpy() if is_torch(result.data) else np.asarray(result.data)
    expected = _brute(info.kind, data, tuple(box), base)
    return _matches(res, expected, data.dtype)


# -- the benchmark ----------------------------------------------------------------


@dataclass
class BenchResult:
    algo: str
    extents: tuple
    box: tuple
    monoid: str
    time_ns: float
    op_count: object  # None: not counted on the GPU ("NA" in the CSV)
    sub_count: object
    peak_bytes: int
    verified: str  # "pass", "fail", or "skipped"
    device: str = "host"
    output: Tensor = field(repr=False, default=None)

    @property
    def n_elements(self) -> int:
        return math.prod(self.extents)

    def csv_row(self) -> str:
        n = self.n_elements
        k = math.prod(self.box)
        oplus = "NA" if self.op_count is None else f"{self.op_count / n:.4f}"
        return ",".join([
            self.algo,
            str(len(self.extents)),
            str(n),
            str(k),
            f"{self.time_ns / n:.1f}",
            oplus,
            f"{self.peak_bytes / n:.1f}",
            self.verified,
        ])


def _device_bytes(algo: str, t: Tensor, k) -> int:
    dtype, op, _ = device_operator(t.ops)
    ext = tuple(int(v) for v in t.data.shape)
    es = np.dtype(dtype).itemsize
    ws = _native.workspace_bytes(algo, _DT_NAME[np.dtype(dtype)], op, ext, k, modulus_of(t.ops))
    return 2 * math.prod(ext) * es + ws


def run_benchmark(
    algo: str,
    extents=None,
    box=None,
    monoid: str = "add-i64",
    seed: int = 0,
    trials: int = 3,
    delay_ns: int = 0,
    verify: bool = False,
    cache: int = 1,
    device: str = "host",
) -> BenchResult:
    """Run one registry entry on one instance; median over ``trials`` runs
    (bench.py:168-234).  ``delay_ns`` is accepted for CLI compatibility and
    must be 0: the device operator cannot be slowed per application."""
    info = resolve_algorithm(algo)
    base_ops = resolve_monoid(monoid)
    if trials < 1:
        raise ConfigurationError(f"trials must be >= 1, got {trials}")
    if delay_ns < 0:
        raise ConfigurationError(f"delay must be >= 0, got {delay_ns}")
    if delay_ns:
        raise ConfigurationError("--delay-ns instruments a CPU operator; the B200 routes have none")
    if device not in ("host", "cuda"):
        raise ConfigurationError(f"device must be 'host' or 'cuda', got {device!r}")
    if extents is None:
        raise UsageError("extents are required")
    if box is None:
        raise UsageError("a box is required")
    check_algorithm_config(info, base_ops)  # monoid mismatch: fail before any work
    check_algorithm_config(info, base_ops, len(validate_extents(extents)))
    t_base = generate_input(base_ops, extents, seed)
    check_algorithm_config(info, base_ops, t_base.data.ndim)
    k = normalize_box(t_base.data.shape, box)

    t = t_base
    sync = lambda: None  # noqa: E731
    if device == "cuda":
        import torch

        t = Tensor(base_ops, torch.from_numpy(np.ascontiguousarray(t_base.data)).cuda())
        sync = torch.cuda.synchronize
    info.run(t, k, cache)  # warm-up: library load, workspace and host-buffer caches
    sync()
    times = []
    result = None
    for _ in range(trials):
        sync()
        start = time.perf_counter_ns()
        result = info.run(t, k, cache)
        sync()
        times.append(time.perf_counter_ns() - start)

    verified = "skipped"
    if verify and t_base.data.size <= VERIFY_ELEMENT_CAP:
        verified = "pass" if verify_against_oracle(info, t_base, k, result) else "fail"
    return BenchResult(
        algo=algo,
        extents=tuple(int(v) for v in t_base.data.shape),
        box=k,
        monoid=base_ops.name,
        time_ns=statistics.median(times),
        op_count=None,
        sub_count=None,
        peak_bytes=_device_bytes(algo, t_base, k),
        verified=verified,
        device=device,
        output=result,
    )


def sweep_extents(d: int, target_elements: int) -> tuple:
    """Near-isotropic extents whose product approximates the target (bench.py:237-242)."""
    if d < 1:
        raise ConfigurationError(f"dimensionality must be >= 1, got {d}")
    side = max(2, round(target_elements ** (1.0 / d)))
    return (side,) * d


def run_sweep(algos, dims, target_elements: int = 1 << 18, box_extent: int = 2,
              monoid: str = "add-i64", seed: int = 0, trials: int = 3, delay_ns: int = 0,
              cache: int = 1, device: str = "host"):
    """One BenchResult per (dimension, algorithm) at a near-constant element
    count (bench.py:245-263)."""
    for d in dims:
        extents = sweep_extents(d, target_elements)
        box = (box_extent,) * d
        for algo in algos:
            yield run_benchmark(algo, extents=extents, box=box, monoid=monoid, seed=seed,
                                trials=trials, delay_ns=delay_ns, cache=cache, device=device)


__all__ = ["ALGORITHMS", "BenchResult", "CSV_HEADER", "FLOAT_RTOL", "VERIFY_ELEMENT_CAP",
           "generate_input", "run_benchmark", "run_sweep", "sweep_extents",
           "verify_against_oracle"]
