"""Pin the CPU oracle to the reference (CPU only, no GPU).

The oracle (oracle/exsum_oracle.c) must reproduce the reference bit for bit on
every golden vector -- floats included, because it keeps the reference's
association -- and agree with the brute-force oracle restatement.
"""

import numpy as np
import pytest

from golden_data import (MONO_OP, corner_cases, ext_cases, load, medium_cases, mono_op,
                         small_cases)
from oracle import oracle as orc


def test_worked_example():
    z = load("kat")
    a, box = z["worked/in"], tuple(z["worked/box"])
    assert np.array_equal(orc.bdbs_included(a, box), z["worked/bdbs"])
    assert np.array_equal(orc.bdbs_excluded(a, box), z["worked/bdbsc"])
    assert np.array_equal(orc.box_complement_excluded(a, box), z["worked/box-complement"])
    assert np.array_equal(orc.box_complement_excluded(a, box, "max"), z["worked/box-complement-max"])
    assert np.array_equal(orc.bdbs_included(a, box, "max"), z["worked/bdbs-max"])
    # total = 91, excluded = total - included (worked_example.py:3-5)
    assert int(z["worked/bdbsc"][0, 0]) == 91 - int(z["worked/bdbs"][0, 0])


def test_frozen_1d_window():
    z = load("kat")
    assert orc.bdbs_included(z["win1d/in"], (4,)).tolist() == [10, 14, 18, 22, 26, 21, 15, 8]
    assert np.array_equal(orc.bdbs_included(z["win1d/in"], (4,)), z["win1d/out"])


def test_exhaustive_1d():
    z = load("kat")
    off = 0
    for n, k in zip(z["ex1d/n"], z["ex1d/k"]):
        vals = z["ex1d/in"][off:off + n]
        assert np.array_equal(orc.bdbs_included(vals, (k,)), z["ex1d/add"][off:off + n])
        assert np.array_equal(orc.bdbs_included(vals, (k,), "max"), z["ex1d/max"][off:off + n])
        off += n


def test_small_random_bit_exact():
    count = 0
    for ci, ext, box, ins, outs in small_cases():
        for key, want in outs.items():
            parts = key.split("/")
            if len(parts) != 2 or parts[1] not in orc.ROUTES:
                continue
            mono, route = parts
            got = orc.ROUTES[route](ins[mono].reshape(ext), box, MONO_OP[mono])
            assert got.dtype == want.dtype
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (ci, key, ext, box)
            count += 1
        for mono in ("add-i64", "max-i64"):
            a = ins[mono].reshape(ext)
            op = MONO_OP[mono]
            assert np.array_equal(orc.brute_included(a, box, op).reshape(-1), outs[f"{mono}/oracle_inc"])
            assert np.array_equal(orc.brute_excluded(a, box, op).reshape(-1), outs[f"{mono}/oracle_exc"])
    assert count >= 1000


def test_medium_bit_exact():
    n = 0
    for m in medium_cases():
        got = orc.ROUTES[m["route"]](m["in"], tuple(m["box"]), MONO_OP[m["mono"]])
        assert np.array_equal(got.view(np.uint8), m["out"].view(np.uint8)), m["key"]
        n += 1
    assert n >= 20


def test_python_brute_force_matches_c():
    rng = np.random.default_rng(5)
    for _ in range(20):
        d = int(rng.integers(1, 4))
        ext = tuple(int(v) for v in rng.integers(1, 5, size=d))
        box = tuple(int(v) for v in rng.integers(1, 6, size=d))
        k = tuple(min(a, b) for a, b in zip(box, ext))
        a = rng.integers(-9, 9, size=ext).astype(np.int64)
        flat = [int(v) for v in a.reshape(-1)]
        for op, ident in (("add", 0), ("max", int(np.iinfo(np.int64).min))):
            assert orc.py_brute_included(ext, flat, k, op, ident) == orc.brute_included(a, box, op).reshape(-1).tolist()
            assert orc.py_brute_excluded(ext, flat, k, op, ident) == orc.brute_excluded(a, box, op).reshape(-1).tolist()


def test_thread_count_does_not_change_bits():
    rng = np.random.default_rng(9)
    a = rng.standard_normal((17, 33, 29))
    for route in ("bdbs", "bdbsc", "box-complement"):
        r1 = orc.ROUTES[route](a, (4, 5, 6), "add", 1)
        r8 = orc.ROUTES[route](a, (4, 5, 6), "add", 8)
        assert np.array_equal(r1, r8)


def test_int64_wraps_like_numpy():
    a = np.array([2**62, 2**62, 2**62, 5], dtype=np.int64)
    got = orc.bdbs_included(a, (3,))
    with np.errstate(over="ignore"):
        want = np.array([a[0] + a[1] + a[2], a[1] + a[2] + a[3], a[2] + a[3], a[3]], dtype=np.int64)
    assert np.array_equal(got, want)


def test_max_rejected_for_weak_route():
    with pytest.raises(orc.OracleError):
        orc.bdbs_excluded(np.zeros((3, 3), dtype=np.int64), (2, 2), "max")


def test_ext_sat_and_mod_add_bit_exact():
    """sat / satc (included.py:37-121, excluded.py:83-85) and mod-add:<m>
    (monoid.py:235-286, incl. non-canonical inputs) against the reference."""
    n = 0
    brute = {"oracle_inc": orc.brute_included, "oracle_exc": orc.brute_excluded}
    for m in ext_cases():
        fn = brute.get(m["route"]) or orc.ROUTES[m["route"]]
        got = fn(m["in"], tuple(m["box"]), mono_op(m["mono"]))
        assert got.dtype == m["out"].dtype
        assert np.array_equal(got.view(np.uint8), m["out"].view(np.uint8)), m["key"]
        n += 1
    assert n >= 1000


def test_corners_bit_exact():
    """corners / corners-spine (excluded.py:191-292) against the reference."""
    n = 0
    for m in corner_cases():
        got = orc.corners_excluded(m["in"], tuple(m["box"]), mono_op(m["mono"]))
        assert np.array_equal(got.view(np.uint8), m["out"].view(np.uint8)), m["tag"]
        n += 1
    assert n >= 50
