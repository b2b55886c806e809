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

    def box_complement(self, R, box):
        return torch.from_numpy(orc.box_complement_excluded(R.numpy(), tuple(box), self.op))
