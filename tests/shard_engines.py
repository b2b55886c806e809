"""CPU stand-in for sharded.CudaEngine built on the oracle (test infrastructure).

It implements the same stage semantics as the C-ABI stage entry points, so the
gloo tests exercise the real orchestration (slab plan, halo exchange, gathers,
rank-order totals, tail slicing) with the checker in place of the kernels.
"""

import numpy as np
import torch

from oracle import oracle as orc


class OracleEngine:
    def __init__(self, op, dtype_name):
        self.op = op
        self.dtype_name = dtype_name

    def axis0(self, x_ext, n_out, box, extra_kind, out=None, extra=None):
        extra_out = extra
        a = x_ext.contiguous().numpy()
        y = orc.windowed_pass(a, 0, min(box[0], a.shape[0]), self.op)[:n_out]
        extra = None
        own = a[:n_out]
        if extra_kind == 1:
            extra = own.max(axis=-1) if self.op == "max" else own.sum(axis=-1, dtype=own.dtype)
            extra = torch.from_numpy(np.ascontiguousarray(extra))
        elif extra_kind == 2:
            if own.dtype.kind == "i":
                with np.errstate(over="ignore"):
                    extra = torch.tensor([int(own.sum(dtype=np.int64))], dtype=torch.int64)
            else:
                extra = torch.tensor([float(own.astype(np.float64).sum())], dtype=torch.float64)
        y = torch.from_numpy(np.ascontiguousarray(y))
        if out is not None:  # write into the caller's views, like the CUDA engine
            out.copy_(y)
            y = out
        if extra_out is not None and extra is not None and extra_kind == 1:
            extra_out.copy_(extra)
            extra = extra_out
        return y, extra

    def bdbs_finish(self, y, box, total):
        a = y.numpy()
        for ax in range(1, a.ndim):
            a = orc.windowed_pass(a, ax, min(box[ax], a.shape[ax]), self.op)
        if total is not None:
            t = total.reshape(-1)[0].item()
            if a.dtype.kind == "i":
                with np.errstate(over="ignore"):
                    a = (np.int64(t) - a).astype(np.int64)
            else:
                a = (a.dtype.type(t) - a).astype(a.dtype)
        return torch.from_numpy(np.ascontiguousarray(a))

    def bc_finish(self, y, box, tail):
        a = y.numpy()
        d = a.ndim
        for ax in range(1, d - 1):
            a = orc.windowed_pass(a, ax, min(box[ax], a.shape[ax]), self.op)
        n = a.shape[-1]
        k = min(box[-1], n)
        acc = np.maximum.accumulate if self.op == "max" else np.add.accumulate
        ident = np.iinfo(np.int64).min if self.op == "max" else a.dtype.type(0)
        P = acc(a, axis=-1)
        S = acc(a[..., ::-1], axis=-1)[..., ::-1]
        out = np.full_like(a, ident)
        comb = np.maximum if self.op == "max" else np.add
        with np.errstate(over="ignore"):
            out[..., 1:] = comb(out[..., 1:], P[..., :-1])
            if k < n:
                out[..., : n - k] = comb(out[..., : n - k], S[..., k:])
            out = comb(out, tail.numpy()[..., None])
        return torch.from_numpy(np.ascontiguousarray(out))

    # the per-shard tail of a 3-D box-complement (sharded.CudaEngine.bc_tail_*)
    def bc_tail_ok(self, ext, k):
        return len(ext) == 2

    def bc_tail_r2(self, R_own, ext, k):
        a = R_own.contiguous().numpy()
        red = a.max(axis=-1) if self.op == "max" else a.sum(axis=-1, dtype=a.dtype)
        return torch.from_numpy(np.ascontiguousarray(red))

    def bc_tail_rows(self, R_ext, R2, ext, k, x0, n_own):
        """T rows [x0, x0+n_own) of BC(R): T1 from R2 (1-D excluded window),
        the window of R along axis 0, its row round along axis 1."""
        n0, n1 = ext
        k0, k1 = min(k[0], n0), min(k[1], n1)
        Rx = R_ext.contiguous().numpy()
        r2 = R2.contiguous().numpy()
        comb = np.maximum if self.op == "max" else np.add
        ident = np.iinfo(np.int64).min if self.op == "max" else Rx.dtype.type(0)
        out = np.empty((n_own, n1), dtype=Rx.dtype)
        with np.errstate(over="ignore"):
            for i in range(n_own):
                x = x0 + i
                t1 = ident
                for y in list(range(0, x)) + list(range(min(x + k0, n0), n0)):
                    t1 = comb(t1, r2[y])
                w = Rx[i]
                for y in range(x + 1, min(x + k0, n0)):
                    w = comb(w, Rx[y - x0])
                for c in range(n1):
                    v = t1
                    for cc in list(range(0, c)) + list(range(min(c + k1, n1), n1)):
                        v = comb(v, w[cc])
                    out[i, c] = v
        return torch.from_numpy(out)

    # the per-axis marginal form for max (sharded.CudaEngine.idem_*): the
    # rank's marginals of its planes, then its output planes from the global ones
    def idem_ok(self, ext):
        return self.op == "max" and self.dtype_name == "int64" and len(ext) >= 2 and sum(ext) <= 4096

    def idem_marginals(self, x_own, ext, x0):
        a = x_own.contiguous().numpy()
        ident = np.iinfo(np.int64).min
        parts = []
        for ax, n in enumerate(ext):
            m = np.full(n, ident, dtype=np.int64)
            if a.size:
                red = a.max(axis=tuple(i for i in range(a.ndim) if i != ax))
                if ax == 0:
                    m[x0:x0 + a.shape[0]] = red
                else:
                    m[:] = red
            parts.append(m)
        return torch.from_numpy(np.concatenate(parts))

    def idem_write(self, marg, ext, box, x0, n_own):
        m = marg.numpy()
        ident = np.iinfo(np.int64).min
        out = None
        off = 0
        for ax, n in enumerate(ext):
            k = min(box[ax], n)
            M = m[off:off + n]
            off += n
            P = np.maximum.accumulate(M)
            S = np.maximum.accumulate(M[::-1])[::-1]
            F = np.full(n, ident, dtype=np.int64)
            F[1:] = P[:-1]
            if k < n:
                F[: n - k] = np.maximum(F[: n - k], S[k:])
            if ax == 0:
                F = F[x0:x0 + n_own]
            shape = [1] * len(ext)
            shape[ax] = F.shape[0]
            Fb = F.reshape(shape)
            out = Fb if out is None else np.maximum(out, Fb)
        full = np.broadcast_to(out, (n_own,) + tuple(ext[1:]))
        return torch.from_numpy(np.ascontiguousarray(full))

    def box_complement(self, R, box):
        return torch.from_numpy(orc.box_complement_excluded(R.numpy(), tuple(box), self.op))
