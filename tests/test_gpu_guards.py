"""Out-of-bounds write guards (compute-sanitizer is not available on the GPU
pool): every route runs through the C ABI on input, output and workspace
regions embedded in larger buffers whose guard bands hold a sentinel; after the
call the guards (and the whole input, which is const) must be unchanged, and
the output must equal the oracle's."""

import ctypes

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side (32 KB for 8-byte types)
SENT = {np.dtype(np.float32): np.float32(-7.25e30), np.dtype(np.float64): -7.25e300,
        np.dtype(np.int64): np.int64(-0x5A5A5A5A5A5A5A5)}
ROUTES = {"bdbs": 0, "bdbsc": 1, "box-complement": 2, "sat": 3, "satc": 4, "corners": 5}

SHAPES = [
    ((1,), (1,)), ((7,), (3,)), ((100,), (100,)), ((1, 1), (1, 1)), ((3, 5), (2, 9)),
    ((33, 17), (4, 16)), ((5, 256), (3, 7)), ((9, 512), (2, 512)), ((4, 1024), (16, 16)),
    ((64, 3), (17, 2)), ((2, 3, 4), (2, 2, 2)), ((13, 7, 9), (3, 1, 4)), ((5, 8, 256), (4, 4, 4)),
    ((3, 16, 1024), (16, 16, 16)), ((130, 4, 33), (128, 4, 1)), ((6, 6, 6, 6), (2, 3, 1, 6)),
    ((2, 3, 2, 3, 2), (2, 2, 2, 2, 2)), ((300, 2), (37, 1)), ((2, 5000), (1, 600)),
    # round-2 kernels: the tiled pair (window 32, element-granular staging), the TMA
    # tensor pass (k = 128 along a strided axis), the 3-D box-complement tail, row
    # strips wider than the fused pair's templates, trailing cubic blocks, the
    # leading-axis pair
    ((45, 33), (32, 32)), ((3, 70, 200), (1, 32, 32)), ((256, 2, 64), (128, 2, 1)),
    ((40, 24, 256), (8, 8, 8)), ((3, 3000), (2, 16)), ((70, 16, 16), (4, 4, 4)),
    ((28, 28, 32), (4, 4, 1)),
]
# profiler scopes the aligned sweep must reach (every kernel family of the routes)
REQUIRED = {"pass_strided", "pass_rows", "fused_pair", "tile_pair", "idem_scan", "idem_bcast",
            "tail_rows", "tail_group", "block_fused", "outer_pair", "total"}


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _cases():
    for shape, box in SHAPES:
        for mono in ("add-f32", "add-f64", "add-i64", "max-i64", "mod-add:97"):
            for route in ROUTES:
                if mono == "max-i64" and route in ("bdbsc", "sat", "satc"):
                    continue
                if route == "corners" and len(shape) not in (2, 3):
                    continue
                yield shape, box, mono, route


@pytest.mark.parametrize("shift", [0, 1])
def test_no_writes_outside_the_call_regions(ex, shift):
    """shift = 1 places every region one element off 16-byte alignment (the
    vectorised kernels must fall back, not fail or fault)."""
    import torch

    from paper_2106_00124_b200 import _native

    L = _native.load()
    rng = np.random.default_rng(31)
    count = 0
    _native.profile_enable(True)
    seen = set()
    for shape, box, mono, route in _cases():
        dt = np.dtype(np.float32 if mono == "add-f32" else np.float64 if mono == "add-f64"
                      else np.int64)
        op = {"max-i64": 1}.get(mono, 2 if mono.startswith("mod-add") else 0)
        m = int(mono.split(":")[1]) if mono.startswith("mod-add") else 0
        dcode = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int64): 2}[dt]
        n = int(np.prod(shape))
        a = (rng.standard_normal(shape).astype(dt) if dt.kind == "f"
             else rng.integers(-1000, 1000, size=shape, dtype=np.int64))
        tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
               np.dtype(np.int64): torch.int64}[dt]
        sent = SENT[dt]
        ext = _native.i64_array(shape)
        bx = _native.i64_array(box)
        wsb = ctypes.c_size_t(0)
        _native.check(L.exsum_route_workspace_bytes(ROUTES[route], dcode, op, m, len(shape), ext,
                                                    bx, ctypes.byref(wsb)))
        # input / output / workspace regions inside guarded buffers (16-byte aligned offsets)
        host_in = np.full(n + 2 * GUARD, sent, dtype=dt)
        host_in[GUARD + shift:GUARD + shift + n] = a.reshape(-1)
        din = torch.from_numpy(host_in).cuda()
        dout = torch.full((n + 2 * GUARD,), float(sent) if dt.kind == "f" else int(sent),
                          dtype=tdt, device="cuda")
        wsn = int(wsb.value)
        dws = torch.full((wsn + 2 * GUARD * 8,), 0xA5, dtype=torch.uint8, device="cuda")
        es = dt.itemsize
        rc = L.exsum_route(ROUTES[route], din.data_ptr() + GUARD * es, dout.data_ptr() + GUARD * es,
                           dcode, op, m, len(shape), ext, bx, dws.data_ptr() + GUARD * 8, wsn,
                           torch.cuda.current_stream().cuda_stream) if not shift else \
            L.exsum_route(ROUTES[route], din.data_ptr() + (GUARD + 1) * es,
                          dout.data_ptr() + (GUARD + 1) * es, dcode, op, m, len(shape), ext, bx,
                          dws.data_ptr() + GUARD * 8, wsn, torch.cuda.current_stream().cuda_stream)
        _native.check(rc)
        torch.cuda.synchronize()
        seen.update(n for n, _, _ in _native.profile_records())
        _native.profile_enable(True)  # clears the records
        h_out = dout.cpu().numpy()
        assert np.array_equal(din.cpu().numpy().view(np.uint8), host_in.view(np.uint8)), \
            ("input modified", shape, box, mono, route)
        lo, hi = GUARD + shift, GUARD + shift + n
        assert np.array_equal(h_out[:lo].view(np.uint8), np.full(lo, sent, dt).view(np.uint8)) \
            and np.array_equal(h_out[hi:].view(np.uint8),
                               np.full(len(h_out) - hi, sent, dt).view(np.uint8)), \
            ("output guard written", shape, box, mono, route)
        w = dws.cpu().numpy()
        assert np.all(w[:GUARD * 8] == 0xA5) and np.all(w[GUARD * 8 + wsn:] == 0xA5), \
            ("workspace guard written", shape, box, mono, route)
        oop = "max" if op == 1 else mono if op == 2 else "add"
        want = orc.ROUTES[route](a.astype(np.float64) if dt.kind == "f" else a, box, oop)
        got = h_out[lo:hi].reshape(shape)
        if dt.kind == "f":
            scale = np.abs(a.astype(np.float64)).sum() * (2 ** len(shape) + 1)
            tol = (sum(shape) + 2 * sum(box) + 2 ** len(shape) + 16) * np.finfo(dt).eps * scale
            assert np.all(np.abs(got.astype(np.float64) - want) <= tol + 1e-300), \
                (shape, box, mono, route)
        else:
            assert np.array_equal(got, want), (shape, box, mono, route)
        count += 1
    _native.profile_enable(False)
    assert count > 300
    if not shift:
        print("scopes:", sorted(seen))
        assert REQUIRED <= seen, sorted(REQUIRED - seen)


def test_building_block_guards(ex):
    """exsum_scan_axis / exsum_add_contribution / exsum_elementwise / exsum_fold
    on guarded, aligned and misaligned regions."""
    import torch

    from paper_2106_00124_b200 import _native

    L = _native.load()
    rng = np.random.default_rng(32)
    st = torch.cuda.current_stream().cuda_stream
    for shape in [(7,), (5, 9), (3, 300, 2), (2, 5000), (4, 6, 10)]:
        n = int(np.prod(shape))
        for dcode, dt, op, m in [(0, np.float32, 0, 0), (1, np.float64, 0, 0), (2, np.int64, 0, 0),
                                 (2, np.int64, 1, 0), (2, np.int64, 2, 97)]:
            for shift in (0, 1):
                a = (rng.standard_normal(shape).astype(dt) if np.dtype(dt).kind == "f"
                     else rng.integers(-1000, 1000, size=shape, dtype=np.int64))
                es = np.dtype(dt).itemsize
                base = np.zeros(n + 2 * GUARD, dtype=dt)
                base[GUARD + shift:GUARD + shift + n] = a.reshape(-1)
                buf = torch.from_numpy(base).cuda()
                ptr = buf.data_ptr() + (GUARD + shift) * es
                ext = _native.i64_array(shape)
                for axis in range(len(shape)):
                    need = ctypes.c_size_t(0)
                    _native.check(L.exsum_scan_workspace_bytes(dcode, op, m, len(shape), ext, axis,
                                                               ctypes.byref(need)))
                    ws = torch.full((int(need.value) + 2 * 4096,), 0x5A, dtype=torch.uint8,
                                    device="cuda")
                    _native.check(L.exsum_scan_axis(ptr, ptr, dcode, op, m, len(shape), ext, axis,
                                                    axis % 2, ws.data_ptr() + 4096,
                                                    int(need.value), st))
                    w = ws.cpu().numpy()
                    assert np.all(w[:4096] == 0x5A) and np.all(w[4096 + int(need.value):] == 0x5A)
                if op != 1:
                    sc = np.array([3], dtype=dt)
                    _native.check(L.exsum_elementwise(ptr, None, sc.ctypes.data, dcode, op, m, 2, n,
                                                      st))
                _native.check(L.exsum_elementwise(ptr, ptr, None, dcode, op, m, 0, n, st))
                res = torch.zeros(2, dtype=buf.dtype, device="cuda")
                fws = torch.empty(int(L.exsum_fold_workspace_bytes()), dtype=torch.uint8,
                                  device="cuda")
                _native.check(L.exsum_fold(ptr, res.data_ptr(), dcode, op, m, n, fws.data_ptr(),
                                           fws.numel(), st))
                torch.cuda.synchronize()
                h = buf.cpu().numpy()
                assert np.array_equal(h[:GUARD + shift].view(np.uint8),
                                      np.zeros(GUARD + shift, dt).view(np.uint8))
                assert np.array_equal(h[GUARD + shift + n:].view(np.uint8),
                                      np.zeros(len(h) - GUARD - shift - n, dt).view(np.uint8))
                assert res[1].item() == 0  # fold writes exactly one element


def test_concurrent_calls_on_separate_streams(ex):
    """Several host threads, one stream each, different routes at once: same
    results as one at a time (host caches, smem-limit cache and the launch
    counters are thread-safe; ctypes releases the GIL)."""
    import threading

    import torch

    rng = np.random.default_rng(33)
    jobs = []
    for i in range(6):
        shape = [(48, 40, 256), (30, 64, 512), (200, 300), (16, 17, 1024), (9, 8, 7, 6), (500,)][i]
        box = [(8, 8, 8), (4, 4, 4), (16, 16), (16, 16, 16), (2, 3, 4, 5), (33,)][i]
        a = torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).cuda()
        route = ["box-complement", "bdbsc", "sat", "bdbs", "box-complement", "bdbs"][i]
        jobs.append((route, a, box))
    fns = {"bdbs": ex.bdbs_included, "bdbsc": ex.bdbs_excluded,
           "box-complement": ex.box_complement_excluded, "sat": ex.sat_included}
    want = [fns[r](ex.Tensor(ex.Float32AddOps(), a), box).data.clone() for r, a, box in jobs]
    torch.cuda.synchronize()
    got = [None] * len(jobs)
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            r, a, box = jobs[i]
            with torch.cuda.stream(s):
                for _ in range(5):
                    got[i] = fns[r](ex.Tensor(ex.Float32AddOps(), a), box).data
            s.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for g, w in zip(got, want):
        assert torch.equal(g, w)
