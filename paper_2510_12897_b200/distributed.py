"""Communication of sharded scenario batches (north_star: "NCCL
over NVLink used only to reduce the shared objective and linking-constraint
terms").

A shard (``sharding.mpopf_shard`` periods, ``scopf.scopf_shard`` N-1
instances) owns the records of its periods/instances and holds, besides its
own variables, copies of the few variables its linking rows read from other
shards: the next period's generator outputs (ramp rows, ``opf.py:468-479``),
the previous period's storage energy (SoC chain, ``opf.py:585-597``), or the
base case's generator outputs (N-1 linking rows ``pg_k - pg_0``).  With those
copies current, cons / jac / hess of a shard need no communication at all.

:class:`ShardComm` is the per-rank plan, computed from the shard windows and
the shard's own plan (no global model), plus one collective at setup:

* :meth:`ShardComm.exchange` -- refresh the borrowed variables from their
  owners: one batched point-to-point round (``torch.distributed``
  ``batch_isend_irecv``; NCCL over NVLink for CUDA tensors, gloo for CPU
  tensors), only the variables some local term actually reads;
* :meth:`ShardComm.objective` -- the shard's partial objective (generated
  kernels, :func:`autodiff.eval_objective`) all-gathered and summed in rank
  order, so every rank gets the same bits run after run (no reduction-order
  nondeterminism);
* gradients need no collective: objective records live on the owner of their
  period/instance, so each owned gradient entry is complete locally.
"""

from __future__ import annotations

import numpy as np

from .core import ModelError


def _owner_of(windows, t: int) -> int:
    for r, (c0, c1) in enumerate(windows):
        if c0 <= t < c1:
            return r
    raise ModelError(f"period/instance {t} is not owned by any shard")


class ShardComm:
    """Exchange plan of rank ``rank``'s shard.

    ``local_periods(r)`` returns the periods/instances (global ids, in local
    order) whose variables shard ``r`` holds; ``windows[r] = (c0, c1)`` the ones
    it owns.  Variable blocks are registered identically on every shard:
    static blocks (no period axis) are replicated, grid blocks ``(n, T)`` hold
    columns ``local_periods(r)`` (``flat = i * Tv + j``, ``core.py:71-73``).

    This rank borrows exactly the entries its terms read whose period another
    shard owns (``self.recv[owner]``: local ids); :meth:`setup` tells each
    owner which of ITS local ids to send (one collective at plan time)."""

    def __init__(self, model, windows, local_periods, rank: int):
        self.model = model
        self.windows = [tuple(map(int, w)) for w in windows]
        self.rank = int(rank)
        self.world = len(self.windows)
        per = [np.asarray(local_periods(r), dtype=np.int64) for r in range(self.world)]
        blocks = [(b.shape[0], len(b.shape) > 1) for b in model.variables]
        if any(g and model.variables[k].shape[1] != per[self.rank].size for k, (_, g) in enumerate(blocks)):
            raise ModelError("shard grid blocks do not match its period list")

        def offsets(r):
            off, out = 0, []
            for n, grid in blocks:
                out.append(off)
                off += n * (per[r].size if grid else 1)
            return out

        mine, offs = per[self.rank], offsets(self.rank)
        used = np.zeros(model.nvar, dtype=bool)
        for tp in model.plan.obj_terms + model.plan.con_terms:
            for cols in tp.cols:
                used[np.asarray(cols, dtype=np.int64)] = True
        recv, need = {}, {}
        for j, t in enumerate(mine.tolist()):
            o = _owner_of(self.windows, t)
            if o == self.rank:
                continue
            pos_o = {int(u): jj for jj, u in enumerate(per[o])}
            if t not in pos_o:
                raise ModelError(f"shard {o} owns period {t} but does not hold it")
            oo = offsets(o)
            for k, (n, grid) in enumerate(blocks):
                if not grid:
                    continue
                i = np.arange(n, dtype=np.int64)
                loc = offs[k] + i * mine.size + j
                keep = used[loc]
                if keep.any():
                    recv.setdefault(o, []).append(loc[keep])
                    need.setdefault(o, []).append((oo[k] + i * per[o].size + pos_o[t])[keep])
        self.recv = {o: np.concatenate(v) for o, v in recv.items()}
        self._need = {o: np.concatenate(v) for o, v in need.items()}
        self.send: dict = {}

    def setup(self, group=None) -> "ShardComm":
        """One collective at plan time: every owner learns which of its local
        variables each borrower reads."""
        import torch.distributed as dist

        needs = [None] * self.world
        dist.all_gather_object(needs, self._need, group=group)
        self.send = {r: np.asarray(nd[self.rank]) for r, nd in enumerate(needs)
                     if r != self.rank and self.rank in nd}
        self._setup_done = True
        return self

    # ------------------------------------------------------------------ comms
    def halo_doubles(self) -> int:
        """Doubles this rank receives per exchange."""
        return int(sum(v.size for v in self.recv.values()))

    def exchange(self, x_local, group=None):
        """Refresh the borrowed variables of ``x_local`` (torch tensor on this
        rank's device, or CPU for gloo) from their owners, in place."""
        import torch
        import torch.distributed as dist

        if self.world > 1 and not getattr(self, "_setup_done", False):
            raise ModelError("ShardComm.setup() must run (collectively) before exchange()")

        ops, bufs = [], []
        dev = x_local.device
        for r, ids in sorted(self.send.items()):
            buf = x_local[torch.as_tensor(ids, device=dev)].contiguous()
            bufs.append(buf)
            ops.append(dist.P2POp(dist.isend, buf, r, group=group))
        rbufs = {}
        for r, ids in sorted(self.recv.items()):
            rb = torch.empty(ids.size, dtype=x_local.dtype, device=dev)
            rbufs[r] = rb
            ops.append(dist.P2POp(dist.irecv, rb, r, group=group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for r, rb in rbufs.items():
            x_local[torch.as_tensor(self.recv[r], device=dev)] = rb
        return x_local

    def reduce_objective(self, partial: float, device=None, group=None) -> float:
        """Sum of the shards' partial objectives, added in rank order on every
        rank (deterministic, identical bits everywhere)."""
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(partial)], dtype=torch.float64, device=device)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=group)
        total = 0.0
        for p in parts:
            total = total + float(p.item())
        return total

    def objective(self, x_local, group=None) -> float:
        """Global objective of the sharded model: this shard's objective on the
        GPU (generated kernels), then :meth:`reduce_objective`."""
        from .autodiff import eval_objective

        dev = x_local.device if getattr(x_local, "is_cuda", False) else None
        return self.reduce_objective(eval_objective(self.model, x_local), device=dev, group=group)


def mpopf_comm(shard, T: int, has_storage: bool, rank: int, n_shards: int) -> ShardComm:
    """Exchange plan of a period shard (``sharding.mpopf_shard``)."""
    from .sharding import period_windows

    windows = period_windows(T, n_shards)

    def local(r):
        c0, c1 = windows[r]
        v0 = c0 - 1 if (has_storage and c0 > 0) else c0
        return np.arange(v0, min(c1 + 1, T))

    return ShardComm(shard.model, windows, local, rank)


def scopf_comm(model, n_instances: int, rank: int, n_shards: int) -> ShardComm:
    """Exchange plan of an N-1 instance shard (``scopf.scopf_shard``): every
    shard holds the base case (instance 0), owned by rank 0."""
    from .scopf import instance_windows

    windows = instance_windows(n_instances, n_shards)

    def local(r):
        c0, c1 = windows[r]
        return np.unique(np.concatenate([[0], np.arange(c0, c1)]))

    return ShardComm(model, windows, local, rank)
