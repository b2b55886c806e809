"""The reference's building blocks on the GPU:
MonoidOps bulk kernels, fold, the reduced-slice scans and add_contribution,
checked against numpy's own semantics (the reference's kernels are numpy
ufuncs, monoid.py:130-286) and composed into box_complement_excluded exactly as
the reference does (excluded.py:129-159)."""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    import torch

    assert torch.cuda.is_available()
    import paper_2106_00124_b200 as ex

    ex._native.load()
    return ex


def _np_accumulate(name, a, axis, reverse):
    w = np.flip(a, axis=axis) if reverse else a
    w = w.copy()
    if name == "max-i64":
        np.maximum.accumulate(w, axis=axis, out=w)
    else:
        np.add.accumulate(w, axis=axis, out=w)
        if name.startswith("mod-add:"):
            np.remainder(w, int(name.split(":")[1]), out=w)
    return np.flip(w, axis=axis).copy() if reverse else w


def _sample(rng, name, shape):
    if name == "add-f64":
        return rng.standard_normal(shape)
    if name == "add-f32":
        return rng.standard_normal(shape).astype(np.float32)
    return rng.integers(-10**6, 10**6, size=shape, dtype=np.int64)


MONOS = ["add-i64", "add-f64", "add-f32", "max-i64", "mod-add:97"]


@pytest.mark.parametrize("name", MONOS)
def test_accumulate_matches_numpy(ex, name):
    import torch

    ops = ex.resolve_monoid(name)
    rng = np.random.default_rng(1)
    for shape in [(7,), (5, 9), (4, 6, 10), (3, 5, 2, 7), (1, 1), (300, 2), (2, 5000)]:
        a = _sample(rng, name, shape)
        for axis in range(len(shape)):
            for rev in (False, True):
                want = _np_accumulate(name, a, axis, rev)
                h = a.copy()
                ops.accumulate(h, axis, reverse=rev)  # numpy in, numpy out (staged)
                d = torch.from_numpy(a.copy()).cuda()
                ops.accumulate(d, axis, reverse=rev)  # device resident
                for got in (h, d.cpu().numpy()):
                    if a.dtype.kind != "f" or shape[axis] < 4096:
                        # sequential per line: numpy's association, bit for bit
                        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), \
                            (shape, axis, rev)
                    else:
                        # too few lines: segmented scan (reassociated), within
                        # n * u of the running magnitude
                        mag = _np_accumulate("add-f64", np.abs(a.astype(np.float64)), axis, rev)
                        tol = shape[axis] * np.finfo(a.dtype).eps * mag
                        assert np.all(np.abs(got.astype(np.float64) - want) <= tol)


@pytest.mark.parametrize("name", MONOS)
def test_elementwise_and_fold(ex, name):
    import math

    ops = ex.resolve_monoid(name)
    rng = np.random.default_rng(2)
    a = _sample(rng, name, (33, 17))
    b = _sample(rng, name, (33, 17))
    m = int(name.split(":")[1]) if name.startswith("mod-add") else 0
    d = a.copy()
    ops.combine_into(d, b)
    want = np.maximum(a, b) if name == "max-i64" else a + b
    if m:
        want = np.remainder(want, m)
    assert np.array_equal(d, want)
    if name == "max-i64":
        with pytest.raises(ex.ConfigurationError):
            ops.subtract_into(a.copy(), b)
        with pytest.raises(ex.ConfigurationError):
            ops.rsubtract_scalar(5, a.copy())
    else:
        d = a.copy()
        ops.subtract_into(d, b)
        want = a - b
        assert np.array_equal(d, np.remainder(want, m) if m else want)
        d = a.copy()
        tot = a.dtype.type(3)
        ops.rsubtract_scalar(tot, d)
        want = tot - a
        assert np.array_equal(d, np.remainder(want, m) if m else want)
    f = ops.fold(a)
    if name == "max-i64":
        assert f == int(a.max())
    elif name == "add-i64":
        assert f == int(a.sum())
    elif m:
        assert f == int(a.sum()) % m
    else:
        exact = math.fsum(a.astype(np.float64).reshape(-1))
        assert abs(f - exact) <= 64 * np.finfo(a.dtype).eps * np.abs(a).sum()
    assert ops.fold(a[:0]) == ops.identity  # empty: the identity
    assert ex.Tensor(ops, a).total_reduce() == f


def test_reduced_slice_helpers(ex):
    rng = np.random.default_rng(3)
    a = rng.integers(-50, 50, size=(4, 5, 6), dtype=np.int64)
    ops = ex.IntAddOps()
    for dim in range(3):
        t = ex.Tensor(ops, a.copy())
        assert np.array_equal(ex.reduced_slice(t, dim), a[tuple(n - 1 for n in a.shape[:dim])])
        ex.prefix_along_dim(t, dim)
        want = a.copy()
        sl = tuple(n - 1 for n in a.shape[:dim])
        want[sl] = np.add.accumulate(a[sl], axis=0)
        assert np.array_equal(t.data, want)
        t = ex.Tensor(ops, a.copy())
        ex.suffix_along_dim(t, dim)
        want = a.copy()
        want[sl] = np.flip(np.add.accumulate(np.flip(a[sl], 0), axis=0), 0)
        assert np.array_equal(t.data, want)
    t = ex.Tensor(ops, a.copy())
    ex.bdbs_along_dim(t, (2, 3, 4), 1, 2)
    want = a.copy()
    want[3] = orc.windowed_pass(a[3], 1, 4)
    assert np.array_equal(t.data, want)
    with pytest.raises(ex.UsageError):
        ex.bdbs_along_dim(t, (2, 3, 4), 2, 1)


def test_add_contribution_matches_reference_semantics(ex):
    rng = np.random.default_rng(4)
    ops = ex.IntAddOps()
    a = rng.integers(-9, 9, size=(3, 4, 5), dtype=np.int64)
    for dim in range(3):
        for off in (-2, -1, 0, 1, 3, 6):
            src = ex.Tensor(ops, a.copy())
            dst = ex.Tensor(ops, np.ones_like(a))
            ex.add_contribution(src, dst, dim, off)
            want = np.ones_like(a)
            red = a[tuple(n - 1 for n in a.shape[:dim])]
            n = a.shape[dim]
            for x in range(n):
                if 0 <= x + off < n:
                    idx = (slice(None),) * dim + (x,)
                    want[idx] += red[x + off]
            assert np.array_equal(dst.data, want), (dim, off)


@pytest.mark.parametrize("name", ["add-i64", "max-i64", "mod-add:11"])
def test_box_complement_composed_from_pieces(ex, name):
    """excluded.py:129-159 written with the GPU pieces equals the fused route."""
    import torch

    ops = ex.resolve_monoid(name)
    rng = np.random.default_rng(5)
    for shape, box in [((6, 7, 5), (2, 3, 2)), ((9, 4), (4, 4)), ((5, 6, 4, 3), (2, 2, 3, 1))]:
        a = rng.integers(-20, 20, size=shape, dtype=np.int64)
        k = ex.normalize_box(shape, box)
        x = torch.from_numpy(a).cuda()
        d = len(shape)
        out = ex.Tensor(ops, torch.full(shape, ops.identity, dtype=torch.int64, device="cuda"))
        cur = ex.Tensor(ops, x.clone())
        nxt = ex.Tensor(ops, torch.empty_like(x))
        win = ex.Tensor(ops, torch.empty_like(x))
        pre = ex.Tensor(ops, torch.empty_like(x))
        for i in range(d):
            live = ex.reduced_slice(cur, i)
            if i < d - 1:
                ex.reduced_slice(nxt, i).copy_(live)
                ex.prefix_along_dim(nxt, i)
            ex.reduced_slice(win, i).copy_(live)
            for j in range(i + 1, d):
                ex.bdbs_along_dim(win, k, i, j)
            ex.reduced_slice(pre, i).copy_(ex.reduced_slice(win, i))
            ex.prefix_along_dim(pre, i)
            ex.add_contribution(pre, out, i, -1)
            ex.suffix_along_dim(win, i)
            ex.add_contribution(win, out, i, k[i])
            if i < d - 1:
                cur, nxt = nxt, cur
        op = "max" if name == "max-i64" else name if name.startswith("mod") else "add"
        want = orc.box_complement_excluded(a, box, op)
        assert np.array_equal(out.data.cpu().numpy(), want), (name, shape)
        route = ex.box_complement_excluded(ex.Tensor(ops, x), box).data.cpu().numpy()
        assert np.array_equal(route, want)
