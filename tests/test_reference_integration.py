"""The drop-in against the real reference harness (CPU; runs where
/root/reference exists, i.e. the build container -- skipped on the GPU box).

register_with_reference() swaps the reference's own registry entries
(bench.py:60-76, the monkeypatch precedent of test_bench.py:243-245); the
reference's harness and CLI then route through the B200 library: its
configuration checks still fire before any work, and without a GPU the call
fails loudly with DeviceError instead of falling back to the CPU."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture
def ref_bench(monkeypatch):
    monkeypatch.syspath_prepend(REF)
    import exsum.bench as bench

    saved = dict(bench.ALGORITHMS)
    yield bench
    bench.ALGORITHMS.clear()
    bench.ALGORITHMS.update(saved)


def test_registry_swap_on_the_real_reference(ref_bench):
    import paper_2106_00124_b200 as ex

    ex.register_with_reference(ref_bench)
    for name in ("sat", "bdbs", "satc", "bdbsc", "box-complement", "corners", "corners-spine"):
        info = ref_bench.ALGORITHMS[name]
        assert isinstance(info, ref_bench.AlgorithmInfo)
        assert info.fn.__module__.startswith("paper_2106_00124_b200"), name
    assert ref_bench.ALGORITHMS["corners"].dims == {2, 3}
    assert ref_bench.ALGORITHMS["corners"].cache_arg == "buffers"
    # routes the B200 build does not accelerate stay the reference's
    assert ref_bench.ALGORITHMS["naive-inc"].fn.__module__.startswith("exsum")


def test_reference_harness_drives_the_gpu_routes(ref_bench):
    import torch

    import paper_2106_00124_b200 as ex
    from exsum.errors import ConfigurationError

    ex.register_with_reference(ref_bench)
    # the reference's own configuration check still runs before any work
    with pytest.raises(ConfigurationError):
        ref_bench.run_benchmark("satc", extents=(6, 6), box=(2, 2), monoid="max-i64")
    if torch.cuda.is_available():
        r = ref_bench.run_benchmark("box-complement", extents=(5, 5), box=(2, 2), seed=3,
                                    verify=True)
        assert r.verified == "pass"
    else:
        # no GPU: a loud failure, never a CPU fallback
        with pytest.raises(ex.DeviceError):
            ref_bench.run_benchmark("box-complement", extents=(5, 5), box=(2, 2), trials=1)
