"""Axis-0 sharding of the box sums across GPUs.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box,
gloo in the CPU tests).  The array is split into contiguous slabs of axis 0
whose boundaries are multiples of the axis-0 window k0, so every rank sees
the same k0-aligned blocks as a single GPU would (float BDBS stays bit-exact).

With the last-axis-first box-complement order (exsum_capi.cu) the only
cross-rank data are:

* the halo: rank r needs the first k0-1 planes of rank r+1 for the axis-0
  windowed pass (windows only look forward);
* BDBSC: the scalar total -- per-rank partials are all-gathered and combined
  in rank order (deterministic; float data folds in float64);
* box-complement: R = fold over the last axis (one value per row, N/n_{d-1}
  elements).  For d = 3 every rank computes only its own rows of the tail
  T = BC(R, k[:-1]): it needs R2 (the fold of R's rows: n0 values, all-gathered)
  and the next rank's first k0-1 rows of R (a halo exchange like the array's);
  otherwise R is all-gathered and every rank computes the whole tail
  redundantly, keeping its own rows.

Everything else (the remaining windowed passes, the row round) is local.

Box-complement with max over int64 (an idempotent operator) takes the
per-axis marginal form instead (csrc/idem_max.cu): every rank folds its own
planes into the sum(ext) marginals, the ranks all-reduce them (elementwise
max), and every rank writes its planes from the global marginals -- no halo
and no tail, one read and one write of each rank's planes.
Per rank at the C4 shape and 8 GPUs: ~1/8 of 4 GiB of HBM traffic per pass vs
a 60 MB halo and a 4 MB all-gather over NVLink.

The orchestration is split into phases (halo, stage 1, combine, stage 2) with
the compute behind an engine: `CudaEngine` calls the C-ABI stage entry points
(exsum_shard_axis0_pass / exsum_bdbs_finish / exsum_box_complement_finish);
the CPU tests plug in an engine built on the oracle to check the decomposition
logic with gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigurationError, UsageError
from .monoid import device_operator
from .tensor import normalize_box

_DT_NAME = {np.dtype(np.float32): "float32", np.dtype(np.float64): "float64",
            np.dtype(np.int64): "int64"}


@dataclass(frozen=True)
class SlabPlan:
    """k0-aligned slabs of axis 0 for `world` ranks."""

    n0: int
    k0: int
    world: int

    def _blocks(self, r):
        nb = math.ceil(self.n0 / self.k0)
        base, extra = divmod(nb, self.world)
        return base + (1 if r < extra else 0)

    def bounds(self, r):
        start_blocks = sum(self._blocks(q) for q in range(r))
        start = min(start_blocks * self.k0, self.n0)
        end = min(start + self._blocks(r) * self.k0, self.n0)
        return start, end

    def halo(self, r):
        """Planes of rank r+1 (and beyond) that rank r needs: min(k0-1, planes left)."""
        _, end = self.bounds(r)
        if end >= self.n0 or end == self.bounds(r)[0]:
            return 0
        return min(self.k0 - 1, self.n0 - end)

    def source_of_halo(self, r):
        """The halo of rank r lives in the next non-empty rank (all of it: slabs hold >= k0 planes)."""
        _, end = self.bounds(r)
        for q in range(r + 1, self.world):
            s, e = self.bounds(q)
            if e > s:
                assert s == end
                return q
        return None


def plan_for(ext, box, world):
    k = normalize_box(ext, box)
    return SlabPlan(int(ext[0]), int(k[0]), int(world)), k


# ---------------------------------------------------------------- engines ----


class CudaEngine:
    """The product path: C-ABI stage entry points on torch CUDA tensors."""

    def __init__(self, ops, device):
        import torch

        self.torch = torch
        self.device = device
        dtype, self.op, self.has_inverse = device_operator(ops)
        self.dtype_name = _DT_NAME[dtype]
        self.L = _native.load()
        self._ws = None

    def _workspace(self, nbytes):
        torch = self.torch
        if self._ws is None or self._ws.numel() < max(nbytes, 1):
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device)
        return self._ws

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def axis0(self, x_ext, n_out, box, extra_kind, out=None, extra=None):
        torch = self.torch
        ext_in = tuple(int(v) for v in x_ext.shape)
        dt, op = _native.DTYPE[self.dtype_name], _native.OP[self.op]
        nbytes = self._ws_bytes(0, ext_in, box, n_out, extra_kind)
        ws = self._workspace(nbytes)
        if out is None:
            out = torch.empty((n_out,) + ext_in[1:], dtype=x_ext.dtype, device=self.device)
        if extra is not None:
            pass
        elif extra_kind == 1:
            extra = torch.empty((n_out,) + ext_in[1:-1], dtype=x_ext.dtype, device=self.device)
        elif extra_kind == 2:
            extra = torch.empty(1, dtype=torch.int64 if self.dtype_name == "int64" else torch.float64,
                                device=self.device)
        _native.check(self.L.exsum_shard_axis0_pass(
            x_ext.data_ptr(), out.data_ptr(), dt, op, len(ext_in), _native.i64_array(ext_in),
            _native.i64_array(box), int(n_out), int(extra_kind),
            extra.data_ptr() if extra is not None else None, ws.data_ptr(), ws.numel(), self._stream()))
        return out, extra

    def bdbs_finish(self, y, box, total, out=None):
        torch = self.torch
        ext = tuple(int(v) for v in y.shape)
        dt, op = _native.DTYPE[self.dtype_name], _native.OP[self.op]
        ws = self._workspace(self._ws_bytes(1, ext, box, 0, 0))
        if out is None:
            out = torch.empty_like(y)
        _native.check(self.L.exsum_bdbs_finish(
            y.data_ptr(), out.data_ptr(), dt, op, len(ext), _native.i64_array(ext),
            _native.i64_array(box), total.data_ptr() if total is not None else None,
            ws.data_ptr(), ws.numel(), self._stream()))
        return out

    def bc_finish(self, y, box, tail, out=None):
        torch = self.torch
        ext = tuple(int(v) for v in y.shape)
        dt, op = _native.DTYPE[self.dtype_name], _native.OP[self.op]
        ws = self._workspace(self._ws_bytes(2, ext, box, 0, 0))
        if out is None:
            out = torch.empty_like(y)
        _native.check(self.L.exsum_box_complement_finish(
            y.data_ptr(), out.data_ptr(), dt, op, len(ext), _native.i64_array(ext),
            _native.i64_array(box), tail.contiguous().data_ptr(), ws.data_ptr(), ws.numel(),
            self._stream()))
        return out

    def bc_tail_ok(self, ext, k):
        """Whether the per-shard tail applies: `ext` / `k` are R's extents and
        box, i.e. the array's without the last axis, and R must be 2-D (a 3-D
        array: R is n0 x n1)."""
        if len(ext) != 2:
            return False
        rc = self.L.exsum_shard_bc_tail(-1, None, None, None, _native.DTYPE[self.dtype_name],
                                         _native.OP[self.op], int(ext[0]), int(ext[1]), int(k[0]),
                                         int(k[1]), 0, 0, None)
        return rc == 0

    def bc_tail_r2(self, R_own, ext, k):
        """The fold of each of this rank's R rows (n_own values)."""
        torch = self.torch
        n_own = int(R_own.shape[0])
        r2 = torch.empty(n_own, dtype=R_own.dtype, device=self.device)
        _native.check(self.L.exsum_shard_bc_tail(
            0, R_own.contiguous().data_ptr() if n_own else None, None,
            r2.data_ptr() if n_own else None, _native.DTYPE[self.dtype_name], _native.OP[self.op],
            int(ext[0]), int(ext[1]), int(k[0]), int(k[1]), 0, n_own, self._stream()))
        return r2

    def bc_tail_rows(self, R_ext, R2, ext, k, x0, n_own):
        """This rank's rows of the tail T = BC(R) from R's rows [x0, x0+n_own+halo)."""
        torch = self.torch
        T = torch.empty((n_own, int(ext[1])), dtype=R_ext.dtype, device=self.device)
        _native.check(self.L.exsum_shard_bc_tail(
            1, R_ext.contiguous().data_ptr() if n_own else None, R2.contiguous().data_ptr(),
            T.data_ptr() if n_own else None, _native.DTYPE[self.dtype_name], _native.OP[self.op],
            int(ext[0]), int(ext[1]), int(k[0]), int(k[1]), int(x0), int(n_own), self._stream()))
        return T

    def idem_ok(self, ext):
        """Whether the per-axis marginal form applies (max over int64, d >= 2,
        sum of the extents within the kernel's tables)."""
        import ctypes

        if self.op != "max":
            return False
        out = ctypes.c_size_t(0)
        rc = self.L.exsum_shard_idem_workspace_bytes(
            _native.DTYPE[self.dtype_name], _native.OP[self.op], len(ext), _native.i64_array(ext),
            ctypes.byref(out))
        self._idem_ws = int(out.value)
        return rc == 0

    def idem_marginals(self, x_own, ext, x0):
        """This rank's marginals (sum(ext) int64; the identity where it holds no element)."""
        torch = self.torch
        S = int(sum(ext))
        marg = torch.empty(S, dtype=torch.int64, device=self.device)
        ws = self._workspace(self._idem_ws)
        n_own = int(x_own.shape[0])
        _native.check(self.L.exsum_shard_idem_marginals(
            x_own.data_ptr() if n_own else None, marg.data_ptr(), _native.DTYPE[self.dtype_name],
            _native.OP[self.op], len(ext), _native.i64_array(ext), int(x0), n_own, ws.data_ptr(),
            ws.numel(), self._stream()))
        return marg

    def idem_write(self, marg, ext, box, x0, n_own):
        torch = self.torch
        out = torch.empty((n_own,) + tuple(ext[1:]), dtype=torch.int64, device=self.device)
        _native.check(self.L.exsum_shard_idem_write(
            marg.data_ptr(), out.data_ptr() if n_own else None, _native.DTYPE[self.dtype_name],
            _native.OP[self.op], len(ext), _native.i64_array(ext), _native.i64_array(box), int(x0),
            int(n_own), self._stream()))
        return out

    def box_complement(self, a, box):
        from .routes import run_device

        ext = tuple(int(v) for v in a.shape)
        return run_device("box-complement", a.contiguous(), self.dtype_name, self.op, ext,
                          normalize_box(ext, box))

    def _ws_bytes(self, stage, ext, box, n_out, extra_kind):
        import ctypes

        out = ctypes.c_size_t(0)
        _native.check(self.L.exsum_shard_workspace_bytes(
            stage, _native.DTYPE[self.dtype_name], _native.OP[self.op], len(ext),
            _native.i64_array(ext), _native.i64_array(box), int(n_out), int(extra_kind),
            ctypes.byref(out)))
        return int(out.value)


# ---------------------------------------------------------- communicator ----


class DistComm:
    """Halo exchange and all-gathers over torch.distributed (NCCL or gloo)."""

    def __init__(self, rank, world, device=None, grouped=True):
        import torch.distributed as dist

        self.dist = dist
        self.rank = rank
        self.world = world
        self.nccl = dist.get_backend() == "nccl"
        self.grouped = grouped

    def exchange_halo(self, plan, x_ext, n_own):
        """Blocking form of start_halo()."""
        for req in self.start_halo(plan, x_ext, n_own):
            req.wait()

    def start_halo(self, plan, x_ext, n_own):
        """Post the halo exchange (send my first halo(r-1) planes to the rank
        whose halo I hold; receive halo(r) planes into x_ext[n_own:]) and
        return the requests; wait() on them before reading the halo."""
        dist = self.dist
        ops = []
        r = self.rank
        # who needs my leading planes: the previous non-empty rank
        prev = None
        for q in range(r - 1, -1, -1):
            s, e = plan.bounds(q)
            if e > s:
                prev = q
                break
        send = None
        if prev is not None and plan.source_of_halo(prev) == r and plan.halo(prev) > 0 and n_own > 0:
            send = x_ext[: plan.halo(prev)].contiguous()
            ops.append(dist.P2POp(dist.isend, send, prev))
        h = plan.halo(r)
        if h > 0:
            src = plan.source_of_halo(r)
            recv = x_ext[n_own:n_own + h]
            ops.append(dist.P2POp(dist.irecv, recv, src))
        if not ops:
            return []
        if self.grouped and self._all_ranks_exchange(plan):
            # every rank takes part (the first and last ranks with one side
            # each): one grouped exchange, posted together (NCCL group)
            return dist.batch_isend_irecv(ops)
        # some rank owns no planes and would post nothing: a grouped call must
        # see every rank, so fall back to plain non-blocking isend / irecv
        return [(dist.isend if o.op is dist.isend else dist.irecv)(o.tensor, o.peer) for o in ops]

    def _all_ranks_exchange(self, plan):
        """True when every rank posts at least one halo send or receive."""
        if self.world < 2:
            return False
        if any(e <= s for s, e in (plan.bounds(q) for q in range(self.world))):
            return False
        return all(plan.halo(q) > 0 for q in range(self.world - 1))

    def all_gather_rows(self, t, counts):
        """Concatenate per-rank tensors of `counts[q]` rows along axis 0."""
        import torch

        dist = self.dist
        m = max(max(counts), 1)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        if t.shape[0] > 0:
            pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad)
        return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)

    def all_gather_scalars(self, t):
        import torch

        bufs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(bufs, t)
        return bufs

    def all_reduce_max(self, t):
        """Elementwise max over the ranks, in place."""
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t


def combine_totals(totals, is_int):
    """Rank-order fold of the per-rank totals (deterministic)."""
    if is_int:
        acc = 0
        for t in totals:
            acc = (acc + int(t.reshape(-1)[0].item())) & ((1 << 64) - 1)
        return acc - (1 << 64) if acc >= 1 << 63 else acc
    acc = 0.0
    for t in totals:
        acc += float(t.reshape(-1)[0].item())
    return acc


# ----------------------------------------------------------- orchestration ----


class ShardedRunner:
    """One rank's share of a sharded route.

    Call with this rank's input slab `x_ext` of shape
    (own planes + halo(rank), *ext[1:]) -- the own planes first, room for the
    halo after them; returns the rank's output planes."""

    def __init__(self, route, ops, ext, box, rank, world, device, comm=None, engine=None):
        if route not in ("bdbs", "bdbsc", "box-complement"):
            raise ConfigurationError(f"unknown route {route!r}")
        dtype, op, has_inverse = device_operator(ops)
        if route == "bdbsc" and not has_inverse:
            raise ConfigurationError(f"algorithm 'bdbsc' requires an invertible monoid")
        if op == "mod-add":
            raise ConfigurationError("the sharded path covers add and max; run mod-add on one GPU")
        self.ext = tuple(int(v) for v in ext)
        if len(self.ext) < 2 and route == "box-complement":
            raise ConfigurationError("sharded box-complement needs d >= 2")
        self.plan, self.k = plan_for(self.ext, box, world)
        self.route, self.rank, self.world = route, rank, world
        self.is_int = np.dtype(dtype).kind == "i"
        self.comm = comm or DistComm(rank, world, device)
        self.engine = engine or CudaEngine(ops, device)
        self.start, self.end = self.plan.bounds(rank)
        self.n_own = self.end - self.start
        self.halo = self.plan.halo(rank)
        # max over int64: the per-axis marginal form -- no halo, no tail
        self.idem = (route == "box-complement" and op == "max" and hasattr(self.engine, "idem_ok")
                     and self.engine.idem_ok(self.ext))
        # 3-D box-complement: each rank computes only its own rows of the tail
        self.own_tail = (route == "box-complement" and not self.idem
                         and hasattr(self.engine, "bc_tail_ok")
                         and self.engine.bc_tail_ok(self.ext[:-1], self.k[:-1]))

    def local_shape(self):
        return (self.n_own + self.halo,) + self.ext[1:]

    def __call__(self, x_ext):
        if tuple(x_ext.shape) != self.local_shape():
            raise UsageError(f"slab shape {tuple(x_ext.shape)} != {self.local_shape()}")
        if self.idem:
            # the halo room (if any) stays unused: the marginal form needs none
            marg = self.engine.idem_marginals(x_ext[:self.n_own], self.ext, self.start)
            marg = self.comm.all_reduce_max(marg)
            return self.engine.idem_write(marg, self.ext, self.k, self.start, self.n_own)
        reqs = self.comm.start_halo(self.plan, x_ext, self.n_own)
        y, extra = self.stage1(x_ext, reqs)
        combined = self.combine(extra, x_ext.device)
        return self.stage2(y, combined)

    def finish(self, x_ext):
        """Stage 1, the combine step and stage 2 (after the halo is in place)."""
        y, extra = self.stage1(x_ext)
        combined = self.combine(extra, x_ext.device)
        return self.stage2(y, combined)

    # -- phases (also driven one virtual rank at a time by run_loopback) --------

    def stage1(self, x_ext, halo_reqs=None):
        """Axis-0 pass of the own planes.  With a halo in flight, the blocks
        that do not need it run first (a standalone pass over the own planes
        is exact for every block but the last, whose stitch partner is the
        halo), then the last block once the halo has landed."""
        extra_kind = {"bdbs": 0, "bdbsc": 2, "box-complement": 1}[self.route]
        if self.n_own == 0:
            for req in halo_reqs or []:
                req.wait()
            return None, None
        k0 = self.k[0]
        split = bool(halo_reqs) and self.halo > 0 and self.n_own >= 2 * k0 and k0 > 1
        if not split:
            for req in halo_reqs or []:
                req.wait()
            return self.engine.axis0(x_ext, self.n_own, self.k, extra_kind)
        import torch

        head = self.n_own - k0
        y = torch.empty((self.n_own,) + self.ext[1:], dtype=x_ext.dtype, device=x_ext.device)
        extra = None
        if extra_kind == 1:
            extra = torch.empty((self.n_own,) + self.ext[1:-1], dtype=x_ext.dtype, device=x_ext.device)
        _, e_a = self.engine.axis0(x_ext[:self.n_own], head, self.k, extra_kind, out=y[:head],
                                   extra=None if extra is None else extra[:head])
        for req in halo_reqs:
            req.wait()
        _, e_b = self.engine.axis0(x_ext[head:], k0, self.k, extra_kind, out=y[head:],
                                   extra=None if extra is None else extra[head:])
        if extra_kind == 2:
            extra = e_a + e_b
        return y, extra

    def local_extra(self, extra, device):
        import torch

        if self.route == "bdbsc" and extra is None:
            return torch.zeros(1, dtype=torch.int64 if self.is_int else torch.float64, device=device)
        if self.route == "box-complement" and extra is None:
            return torch.zeros((0,) + self.ext[1:-1], dtype=_torch_dtype(self.engine), device=device)
        return extra

    def combine(self, extra, device):
        extra = self.local_extra(extra, device)
        if self.route == "bdbsc":
            # stays on the device (no host sync in the step): a fixed-order
            # reduction of the world's partial totals
            import torch

            return torch.stack(self.comm.all_gather_scalars(extra)).sum(dim=0)
        if self.route == "box-complement":
            counts = [self.plan.bounds(q)[1] - self.plan.bounds(q)[0] for q in range(self.world)]
            if self.own_tail:
                return self.own_tail_rows(extra, counts)
            R = self.comm.all_gather_rows(extra, counts)
            return self.engine.box_complement(R, self.k[:-1])  # tail T, computed redundantly
        return None

    def own_tail_rows(self, R_own, counts, R_halo=None):
        """This rank's rows of T: R2 all-gathered (n0 values), the next rank's
        first k0-1 rows of R by the halo exchange (R_halo given: loopback)."""
        import torch

        ext2, k2 = self.ext[:-1], self.k[:-1]
        r2 = self.engine.bc_tail_r2(R_own, ext2, k2)
        R2 = self.comm.all_gather_rows(r2, counts)
        R_ext = torch.empty((self.n_own + self.halo,) + tuple(R_own.shape[1:]), dtype=R_own.dtype,
                            device=R_own.device)
        if self.n_own:
            R_ext[:self.n_own] = R_own
        if R_halo is not None:
            if self.halo:
                R_ext[self.n_own:] = R_halo
        else:
            for req in self.comm.start_halo(self.plan, R_ext, self.n_own):
                req.wait()
        return self.engine.bc_tail_rows(R_ext, R2, ext2, k2, self.start, self.n_own)

    def stage2(self, y, combined):
        if y is None:
            return None
        if self.route == "bdbs":
            return self.engine.bdbs_finish(y, self.k, None)
        if self.route == "bdbsc":
            return self.engine.bdbs_finish(y, self.k, combined.reshape(1).contiguous())
        tail = combined if self.own_tail else combined[self.start:self.end]
        return self.engine.bc_finish(y, self.k, tail)


def _torch_dtype(engine):
    import torch

    return {"float32": torch.float32, "float64": torch.float64, "int64": torch.int64}[
        getattr(engine, "dtype_name", "float64")]


class _LoopbackComm:
    """In-process stand-in for DistComm: every virtual rank's stage-1 outputs
    are already known, so the gathers are concatenations."""

    def __init__(self, world):
        self.world = world
        self.extras = None

    def all_reduce_max(self, t):
        import torch

        return torch.stack(self.extras).amax(dim=0)

    def all_gather_scalars(self, t):
        return self.extras

    def all_gather_rows(self, t, counts):
        import torch

        return torch.cat([e[:c] for e, c in zip(self.extras, counts)], dim=0)


class _Done:
    def wait(self):
        return None


def run_loopback(route, ops, a, box, world, engine, split=True, concat=True):
    """Run the sharded route with `world` virtual ranks in this process (one
    GPU): halos are sliced from the global array, the combine step sees every
    rank's stage-1 output.  Returns the concatenated output.  This exercises
    the same stage entry points and slab arithmetic as the multi-process path.
    concat=False returns the per-rank outputs as a list (no 2 N s concatenation:
    tools/sharded_rank_time.py times the ranks' stages alone)."""
    import torch

    ext = tuple(int(v) for v in a.shape)
    comm = _LoopbackComm(world)
    runners = [ShardedRunner(route, ops, ext, box, r, world, a.device, comm=comm, engine=engine)
               for r in range(world)]
    if runners and runners[0].idem:
        comm.extras = [engine.idem_marginals(a[r.start:r.end].contiguous(), ext, r.start)
                       for r in runners]
        marg = comm.all_reduce_max(None)
        outs = [engine.idem_write(marg, ext, r.k, r.start, r.n_own) for r in runners if r.n_own > 0]
        return torch.cat(outs, dim=0) if concat else outs
    ys, extras = [], []
    for r in runners:
        x_ext = a[r.start:r.end + r.halo]
        # split=True takes the overlap path (interior blocks, then the last one)
        y, e = r.stage1(x_ext.contiguous(), [_Done()] if split and r.halo > 0 else None)
        ys.append(y)
        extras.append(r.local_extra(e, a.device))
    comm.extras = extras
    outs = []
    if runners and runners[0].own_tail:
        counts = [r.n_own for r in runners]
        R_all = torch.cat([e[:c] for e, c in zip(extras, counts)], dim=0)
        comm.extras = [r.engine.bc_tail_r2(e, r.ext[:-1], r.k[:-1]) for r, e in zip(runners, extras)]
        for r, y in zip(runners, ys):
            T = r.own_tail_rows(extras[runners.index(r)], counts, R_halo=R_all[r.end:r.end + r.halo])
            o = r.stage2(y, T)
            if o is not None:
                outs.append(o)
        return torch.cat(outs, dim=0) if concat else outs
    combined = runners[0].combine(extras[0], a.device) if world > 0 else None
    for r, y in zip(runners, ys):
        o = r.stage2(y, combined)
        if o is not None:
            outs.append(o)
    return torch.cat(outs, dim=0) if concat else outs


def make_local_slab(gen_planes, ext, rank, world, box=None):
    """Allocate this rank's slab (own planes + halo room) and fill the own
    planes with gen_planes(p0, p1) -- planes [p0, p1) of the GLOBAL array, so
    the ranks together hold exactly the array one GPU would see (and an N>1
    run can be checked against it).  The halo is filled by the exchange."""
    plan, _ = plan_for(ext, box if box is not None else (1,) * len(ext), world)
    start, end = plan.bounds(rank)
    own = gen_planes(start, end)
    if tuple(own.shape) != (end - start,) + tuple(ext[1:]):
        raise UsageError(f"gen_planes({start}, {end}) returned shape {tuple(own.shape)}")
    halo = plan.halo(rank)
    if halo == 0:
        return own
    import torch

    x = torch.empty((end - start + halo,) + tuple(ext[1:]), dtype=own.dtype, device=own.device)
    x[: end - start] = own
    return x
