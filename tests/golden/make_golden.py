"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--only-ext | --only-corners]

It imports the unmodified reference package read-only from
/root/reference/pkg/src (``exsum``), runs its public entry points
(``bdbs_1d``, ``bdbs_included``, ``bdbs_excluded``, ``box_complement_excluded``
and the brute-force ``oracle_included`` / ``oracle_excluded``) on seeded inputs,
and writes the inputs and outputs to ``tests/golden/*.npz``.  The fixtures are
committed so the GPU box (which has no /root/reference) can check the CUDA path
against them.

float32 is not a reference monoid; as SURVEY.md 8(c) prescribes, a test-side
subclass of the reference's ``FloatAddOps`` with ``dtype=float32`` runs the
unchanged reference code paths.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import exsum  # noqa: F401  (the reference package)

    return exsum


def make():
    ex = _import_reference()

    class AddF32(ex.FloatAddOps):
        name = "add-f32"
        dtype = np.dtype(np.float32)
        identity = np.float32(0.0)

    monoids = {
        "add-i64": ex.IntAddOps(),
        "max-i64": ex.IntMaxOps(),
        "add-f64": ex.FloatAddOps(),
        "add-f32": AddF32(),
    }
    routes = {
        "bdbs": ex.bdbs_included,
        "bdbsc": ex.bdbs_excluded,
        "box-complement": ex.box_complement_excluded,
    }

    def run(route, mono, arr, box):
        ops = monoids[mono]
        t = ex.Tensor(ops, np.ascontiguousarray(arr, dtype=ops.dtype))
        return routes[route](t, box).data.copy()

    # -- 1. known-answer tests -------------------------------------------------
    kat = {}
    # the reference's shared worked example (pkg/tests/worked_example.py), run
    # through the reference rather than copied
    sys.path.insert(0, "/root/reference/pkg/tests")
    import worked_example as we

    a55 = np.array(we.INPUT_5X5, dtype=np.int64)
    kat["worked/in"] = a55
    kat["worked/box"] = np.array(we.BOX, dtype=np.int64)
    kat["worked/bdbs"] = run("bdbs", "add-i64", a55, we.BOX)
    kat["worked/bdbsc"] = run("bdbsc", "add-i64", a55, we.BOX)
    kat["worked/box-complement"] = run("box-complement", "add-i64", a55, we.BOX)
    kat["worked/box-complement-max"] = run("box-complement", "max-i64", a55, we.BOX)
    kat["worked/bdbs-max"] = run("bdbs", "max-i64", a55, we.BOX)
    # frozen 1-D window of test_scan.py:111-112, through bdbs_1d
    kat["win1d/in"] = np.arange(1, 9, dtype=np.int64)
    kat["win1d/out"] = ex.bdbs_1d(monoids["add-i64"], list(range(1, 9)), 4)
    # exhaustive 1-D (test_scan.py:128-135 style): n <= 12, k <= n+2, + and max
    rng = np.random.default_rng(4)
    ex1d_in, ex1d_n, ex1d_k, ex1d_add, ex1d_max = [], [], [], [], []
    for n in range(1, 13):
        for k in range(1, n + 3):
            vals = rng.integers(-50, 50, size=n).astype(np.int64)
            ex1d_in.append(vals)
            ex1d_n.append(n)
            ex1d_k.append(k)
            ex1d_add.append(ex.bdbs_1d(monoids["add-i64"], vals, k))
            ex1d_max.append(ex.bdbs_1d(monoids["max-i64"], vals, k))
    kat["ex1d/in"] = np.concatenate(ex1d_in)
    kat["ex1d/n"] = np.array(ex1d_n, dtype=np.int64)
    kat["ex1d/k"] = np.array(ex1d_k, dtype=np.int64)
    kat["ex1d/add"] = np.concatenate(ex1d_add)
    kat["ex1d/max"] = np.concatenate(ex1d_max)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kat)

    # -- 2. small random instances (acceptance C2 style, test_acceptance.py:93-105)
    # integer values in [0,100) for + and max (oracle-exact), plus the brute
    # force oracle outputs; float instances use rng.random for the float monoids
    def small_cases(seed, plan):
        rng = np.random.default_rng(seed)
        for d, count in plan:
            for _ in range(count):
                while True:
                    ext = tuple(int(v) for v in rng.integers(1, 7, size=d))
                    if d < 4 or int(np.prod(ext)) <= 360:
                        break
                box = tuple(int(rng.integers(1, n + 2)) for n in ext)
                yield ext, box, rng

    small = {"meta": []}
    blobs = {}
    plan = [(1, 30), (2, 40), (3, 40), (4, 20)]
    for ci, (ext, box, rng) in enumerate(small_cases(2024, plan)):
        n = int(np.prod(ext))
        ivals = rng.integers(0, 100, size=ext).astype(np.int64)
        fvals = rng.random(ext)
        small["meta"].append({"ext": ext, "box": box})
        blobs[f"{ci}/int"] = ivals
        blobs[f"{ci}/f64"] = fvals
        clipped = tuple(min(k, m) for k, m in zip(box, ext))
        for mono in ("add-i64", "max-i64"):
            ops = monoids[mono]
            flat = [int(v) for v in ivals.reshape(-1)]
            blobs[f"{ci}/{mono}/oracle_inc"] = np.array(
                ex.oracle_included(ext, flat, clipped, ops.combine, ops.identity), dtype=np.int64)
            blobs[f"{ci}/{mono}/oracle_exc"] = np.array(
                ex.oracle_excluded(ext, flat, clipped, ops.combine, ops.identity), dtype=np.int64)
            for route in routes:
                if route == "bdbsc" and mono == "max-i64":
                    continue
                blobs[f"{ci}/{mono}/{route}"] = run(route, mono, ivals, box)
        for mono in ("add-f64", "add-f32"):
            arr = fvals.astype(monoids[mono].dtype)
            for route in routes:
                blobs[f"{ci}/{mono}/{route}"] = run(route, mono, arr, box)
        assert n <= 360
    blobs["meta"] = np.frombuffer(json.dumps(small["meta"]).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **blobs)

    # -- 3. medium instances shaped like the BASELINE configs (reduced sizes) ---
    # same value distributions as SURVEY 8(d); outputs from the reference.
    med = {}
    meta = []

    def add_case(name, arr, mono, route, box):
        key = f"{name}/{mono}/{route}/{'x'.join(map(str, box))}"
        if f"{name}/in/{mono}" not in med:
            med[f"{name}/in/{mono}"] = np.ascontiguousarray(arr, dtype=monoids[mono].dtype)
        med[key] = run(route, mono, med[f"{name}/in/{mono}"], box)
        meta.append({"key": key, "name": name, "mono": mono, "route": route, "box": list(box),
                     "ext": list(arr.shape)})

    rng = np.random.default_rng(0)
    c1 = rng.random((96, 80))  # C1-like: f64 uniform, k=(32,32)
    add_case("c1", c1, "add-f64", "bdbs", (32, 32))
    rng = np.random.default_rng(0)
    c2 = rng.integers(-2**20, 2**20, size=(24, 20, 28), dtype=np.int64)  # C2-like
    add_case("c2", c2, "max-i64", "box-complement", (8, 8, 8))
    add_case("c2", c2, "add-i64", "bdbsc", (8, 8, 8))
    add_case("c2", c2, "add-i64", "box-complement", (8, 8, 8))
    add_case("c2", c2, "max-i64", "bdbs", (8, 8, 8))
    for shape in [(64, 64), (16, 16, 16), (8, 8, 8, 8), (5, 6, 7, 5, 6), (4, 4, 4, 4, 4, 4)]:
        rng = np.random.default_rng(0)  # C3-like: k=4 everywhere
        name = "c3_" + "x".join(map(str, shape))
        add_case(name, rng.standard_normal(shape, dtype=np.float32), "add-f32", "bdbs",
                 (4,) * len(shape))
        rng = np.random.default_rng(0)
        add_case(name + "_i", rng.integers(-2**20, 2**20, size=shape, dtype=np.int64),
                 "max-i64", "bdbs", (4,) * len(shape))
    rng = np.random.default_rng(0)
    c4 = rng.random((32, 24, 40), dtype=np.float32)  # C4-like f32 uniform, k=16
    add_case("c4", c4, "add-f32", "box-complement", (16, 16, 16))
    add_case("c4", c4, "add-f32", "bdbsc", (16, 16, 16))
    add_case("c4_64", c4.astype(np.float64), "add-f64", "box-complement", (16, 16, 16))
    add_case("c4_64", c4.astype(np.float64), "add-f64", "bdbsc", (16, 16, 16))
    rng = np.random.default_rng(0)
    c5 = rng.standard_normal((36, 20, 28))  # C5-like f64 normal, box sweep
    for box in [(2, 2, 2), (8, 8, 8), (32, 32, 32), (128, 4, 1), (1, 1, 512)]:
        add_case("c5", c5, "add-f64", "bdbs", box)
        add_case("c5", c5, "add-f64", "bdbsc", box)
    med["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "medium.npz"), **med)
    print("wrote kat.npz, small.npz, medium.npz to", HERE)


def make_ext():
    """ext.npz: the section 8(f) rows -- "sat"/"satc" (included.py:37-121,
    excluded.py:83-85) for the invertible monoids and the ``mod-add:<m>``
    monoid (monoid.py:235-286) on every route, through the reference."""
    ex = _import_reference()
    from exsum.excluded import sat_excluded
    from exsum.included import sat_included

    class AddF32(ex.FloatAddOps):
        name = "add-f32"
        dtype = np.dtype(np.float32)
        identity = np.float32(0.0)

    routes = {
        "bdbs": ex.bdbs_included,
        "bdbsc": ex.bdbs_excluded,
        "box-complement": ex.box_complement_excluded,
        "sat": sat_included,
        "satc": sat_excluded,
    }

    def mono(name):
        if name == "add-f32":
            return AddF32()
        return ex.resolve_monoid(name)

    out = {}
    meta = []

    def case(tag, arr, mname, box, route_names):
        ops = mono(mname)
        arr = np.ascontiguousarray(arr, dtype=ops.dtype)
        key_in = f"{tag}/in"
        out[key_in] = arr
        for r in route_names:
            t = ex.Tensor(ops, arr.copy())
            res = routes[r](t, box).data.copy()
            key = f"{tag}/{r}"
            out[key] = res
            meta.append({"key": key, "in": key_in, "mono": mname, "route": r, "box": list(box),
                         "ext": list(arr.shape)})
        if arr.size <= 400 and mname != "add-f32":
            clipped = tuple(min(k, m) for k, m in zip(box, arr.shape))
            flat = [v.item() for v in arr.reshape(-1)]
            for kind, fn in (("inc", ex.oracle_included), ("exc", ex.oracle_excluded)):
                key = f"{tag}/oracle_{kind}"
                out[key] = np.array(fn(arr.shape, flat, clipped, ops.combine, ops.identity),
                                    dtype=ops.dtype).reshape(arr.shape)
                meta.append({"key": key, "in": key_in, "mono": mname, "route": "oracle_" + kind,
                             "box": list(box), "ext": list(arr.shape)})

    rng = np.random.default_rng(2106)
    ci = 0
    # small random instances, d = 1..4, every invertible monoid: sat + satc
    for d, count in [(1, 12), (2, 16), (3, 16), (4, 8)]:
        for _ in range(count):
            while True:
                ext = tuple(int(v) for v in rng.integers(1, 7, size=d))
                if int(np.prod(ext)) <= 360:
                    break
            box = tuple(int(rng.integers(1, n + 2)) for n in ext)
            ivals = rng.integers(0, 100, size=ext).astype(np.int64)
            fvals = rng.random(ext)
            case(f"s{ci}_i", ivals, "add-i64", box, ["sat", "satc"])
            case(f"s{ci}_f", fvals, "add-f64", box, ["sat", "satc"])
            case(f"s{ci}_g", fvals.astype(np.float32), "add-f32", box, ["sat", "satc"])
            ci += 1
    # mod-add: canonical inputs (generate_input style, bench.py:103-114) and
    # non-canonical ones (negative, >= m, large), every route
    mods = [2, 7, 11, 97, 1000003, 2**31]
    every = list(routes)
    for d, count in [(1, 10), (2, 14), (3, 14), (4, 6)]:
        for _ in range(count):
            while True:
                ext = tuple(int(v) for v in rng.integers(1, 7, size=d))
                if int(np.prod(ext)) <= 360:
                    break
            box = tuple(int(rng.integers(1, n + 2)) for n in ext)
            m = mods[ci % len(mods)]
            canon = rng.integers(0, 100, size=ext).astype(np.int64) % m
            case(f"m{ci}_c", canon, f"mod-add:{m}", box, every)
            raw = rng.integers(-3 * m, 3 * m, size=ext).astype(np.int64)
            if ci % 3 == 0:
                raw = raw + rng.integers(-2**40, 2**40, size=ext).astype(np.int64)
            case(f"m{ci}_r", raw, f"mod-add:{m}", box, every)
            ci += 1
    # medium: C-like shapes for sat/satc and mod-add
    r0 = np.random.default_rng(0)
    case("c1sat", r0.random((96, 80)), "add-f64", (32, 32), ["sat", "satc"])
    r0 = np.random.default_rng(0)
    case("c3sat", r0.standard_normal((16, 16, 16), dtype=np.float32), "add-f32", (4, 4, 4),
         ["sat"])
    r0 = np.random.default_rng(0)
    case("c2sat", r0.integers(-2**20, 2**20, size=(24, 20, 28), dtype=np.int64), "add-i64",
         (8, 8, 8), ["sat", "satc"])
    r0 = np.random.default_rng(0)
    case("c5sat", r0.standard_normal((12, 10, 14, 9)), "add-f64", (3, 4, 2, 5), ["sat", "satc"])
    r0 = np.random.default_rng(0)
    case("mmed", r0.integers(0, 100, size=(20, 18, 22), dtype=np.int64) % 97, "mod-add:97",
         (4, 4, 4), every)
    r0 = np.random.default_rng(0)
    case("mmed2", r0.integers(-2**31, 2**31, size=(40, 50), dtype=np.int64), f"mod-add:{2**31}",
         (8, 1), every)
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "ext.npz"), **out)
    print("wrote ext.npz:", len(meta), "outputs")


def make_corners():
    """corners.npz: corners_excluded (every buffer count) and
    corners_spine_excluded (every cache depth), excluded.py:191-292, on 2-D
    and 3-D inputs for every monoid, through the reference."""
    ex = _import_reference()
    from exsum.excluded import corners_excluded, corners_spine_excluded

    class AddF32(ex.FloatAddOps):
        name = "add-f32"
        dtype = np.dtype(np.float32)
        identity = np.float32(0.0)

    def mono(name):
        return AddF32() if name == "add-f32" else ex.resolve_monoid(name)

    out, meta = {}, []
    rng = np.random.default_rng(191)
    monos = ["add-i64", "max-i64", "add-f64", "add-f32", "mod-add:11", "mod-add:2147483648"]
    ci = 0
    for d, count in [(2, 24), (3, 24)]:
        for _ in range(count):
            ext = tuple(int(v) for v in rng.integers(1, 8 if d == 2 else 6, size=d))
            box = tuple(int(rng.integers(1, n + 2)) for n in ext)
            mname = monos[ci % len(monos)]
            ops = mono(mname)
            if ops.dtype.kind == "f":
                arr = rng.random(ext).astype(ops.dtype)
            elif mname.startswith("mod-add"):
                arr = rng.integers(-3 * 11, 3 * 11, size=ext).astype(np.int64)
            else:
                arr = rng.integers(-100, 100, size=ext).astype(np.int64)
            tag = f"k{ci}"
            out[f"{tag}/in"] = arr
            results = []
            for c in range(1, d + 1):
                results.append(corners_excluded(ex.Tensor(ops, arr.copy()), box, buffers=c).data)
                results.append(corners_spine_excluded(ex.Tensor(ops, arr.copy()), box,
                                                      cache_depth=c).data)
            for r in results[1:]:  # every variant agrees bit for bit
                assert r.tobytes() == results[0].tobytes()
            out[f"{tag}/out"] = results[0].copy()
            meta.append({"tag": tag, "mono": mname, "box": list(box), "ext": list(ext)})
            ci += 1
    r0 = np.random.default_rng(0)
    for tag, arr, mname, box in [
        ("c2like", r0.integers(-2**20, 2**20, size=(24, 20, 28), dtype=np.int64), "max-i64",
         (8, 8, 8)),
        ("c4like", r0.random((32, 24, 40), dtype=np.float32), "add-f32", (16, 16, 16)),
        ("c1like", r0.random((96, 80)), "add-f64", (32, 32)),
        ("c2add", r0.integers(-2**20, 2**20, size=(20, 18, 22), dtype=np.int64), "add-i64",
         (4, 5, 3)),
    ]:
        out[f"{tag}/in"] = arr
        out[f"{tag}/out"] = corners_excluded(ex.Tensor(mono(mname), arr.copy()), box).data.copy()
        meta.append({"tag": tag, "mono": mname, "box": list(box), "ext": list(arr.shape)})
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "corners.npz"), **out)
    print("wrote corners.npz:", len(meta), "cases")


if __name__ == "__main__":
    if "--only-ext" in sys.argv:
        make_ext()
    elif "--only-corners" in sys.argv:
        make_corners()
    else:
        make()
        make_ext()
        make_corners()
