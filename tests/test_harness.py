"""The harness mirror: host logic on CPU, the end-to-end
runs on the GPU (marked).  The command line is the reference's own
(`exsum run/sweep` after `register_with_reference()`); this
package ships no CLI of its own."""

import csv
import io

import numpy as np
import pytest

import paper_2106_00124_b200 as ex
from golden_data import ext_cases, small_cases
from paper_2106_00124_b200 import harness


def test_csv_header_matches_reference():
    # bench.py:39 -- scripts written against `exsum run` read the same columns
    assert harness.CSV_HEADER == \
        "algo,d,N,K,time_ns_per_elem,oplus_per_elem,peak_bytes_per_elem,verified"
    r = harness.BenchResult("bdbsc", (6, 6), (2, 2), "add-i64", 3600.0, None, None, 7200,
                            "pass")
    rows = list(csv.reader(io.StringIO(harness.CSV_HEADER + "\n" + r.csv_row())))
    assert rows[1] == ["bdbsc", "2", "36", "4", "100.0", "NA", "200.0", "pass"]


def test_sweep_extents_and_generate_input():
    assert harness.sweep_extents(3, 1 << 18) == (64, 64, 64)
    assert harness.sweep_extents(8, 10) == (2,) * 8
    with pytest.raises(ex.ConfigurationError):
        harness.sweep_extents(0, 100)
    v = harness.generate_input(ex.IntAddOps(), (2, 2), 0).data
    assert np.all((v >= 0) & (v < 100))
    m = harness.generate_input(ex.resolve_monoid("mod-add:7"), (60,), 2).data
    assert np.all((m >= 0) & (m < 7))
    f = harness.generate_input(ex.resolve_monoid("add-f32"), (50,), 1).data
    assert f.dtype == np.float32 and np.all((f >= 0) & (f < 1))


def test_brute_force_matches_reference_oracle():
    """The verifier's fold equals the reference's oracle_included/excluded."""
    n = 0
    for ci, ext, box, ins, outs in small_cases():
        if ci % 4:
            continue
        clipped = tuple(min(k, e) for k, e in zip(box, ext))
        for mono in ("add-i64", "max-i64"):
            a = ins[mono].reshape(ext)
            ops = ex.resolve_monoid(mono)
            got_i = np.array(harness._brute("included", a, clipped, ops), dtype=np.int64)
            got_e = np.array(harness._brute("excluded", a, clipped, ops), dtype=np.int64)
            assert np.array_equal(got_i, outs[f"{mono}/oracle_inc"]), (ci, mono)
            assert np.array_equal(got_e, outs[f"{mono}/oracle_exc"]), (ci, mono)
            n += 1
    for m in ext_cases():
        if m["route"].startswith("oracle_") and m["mono"].startswith("mod-add:") and m["in"].size < 200:
            kind = "included" if m["route"] == "oracle_inc" else "excluded"
            got = harness._brute(kind, m["in"], tuple(m["box"]), ex.resolve_monoid(m["mono"]))
            assert np.array_equal(np.array(got, dtype=np.int64).reshape(m["out"].shape), m["out"])
            n += 1
    assert n >= 40


def test_harness_configuration_errors_before_work():
    # every one of these fails before any device work (no GPU needed), with
    # the reference's exception types (bench.check_algorithm_config)
    for kw in (dict(algo="bdbsc", monoid="max-i64"), dict(algo="sat", monoid="max-i64"),
               dict(algo="bdbs", monoid="mod-add:1"), dict(algo="naive-inc")):
        algo = kw.pop("algo")
        with pytest.raises(ex.ConfigurationError):
            harness.run_benchmark(algo, extents=(4, 4), box=(2, 2), **kw)
    with pytest.raises(ex.UsageError):
        harness.run_benchmark("bdbs", extents=(4, 4), box=(2,))
    with pytest.raises(ex.ConfigurationError):
        harness.run_benchmark("corners", extents=(4,), box=(2,))
    with pytest.raises(ex.ConfigurationError):
        harness.run_benchmark("corners-spine", extents=(4, 4, 4, 4), box=(2, 2, 2, 2))


@pytest.mark.gpu
def test_run_benchmark_verifies_every_route():
    for algo in ("bdbs", "bdbsc", "box-complement", "sat", "satc", "corners", "corners-spine"):
        for mono in ("add-i64", "add-f64", "add-f32", "mod-add:13", "max-i64"):
            if mono == "max-i64" and algo in ("bdbsc", "sat", "satc"):
                continue
            for device in ("host", "cuda"):
                r = harness.run_benchmark(algo, extents=(5, 6, 4), box=(2, 3, 2), monoid=mono,
                                          seed=3, trials=2, verify=True, device=device)
                assert r.verified == "pass", (algo, mono, device)
                assert r.peak_bytes >= 2 * 120 * 4 and r.time_ns > 0


@pytest.mark.gpu
def test_run_sweep_rows():
    rows = list(harness.run_sweep(["bdbs", "box-complement", "sat"], range(1, 5), target_elements=4096,
                             trials=1))
    assert len(rows) == 3 * 4 and all(r.time_ns > 0 for r in rows)
    assert rows[0].csv_row().startswith("bdbs,1,")
    big = harness.run_benchmark("bdbs", extents=(17, 17, 15), box=(4, 4, 4), trials=1,
                                verify=True)
    assert big.verified == "skipped"  # above VERIFY_ELEMENT_CAP, like the reference
