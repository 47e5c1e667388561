"""Scenario-batch sharding across GPUs.

Multi-period AC-OPF (MP96) is sharded by **periods**: rank ``s`` owns the
constraint/objective records of periods ``[c0, c1)`` and holds variables for
``[v0, v1)`` -- one overlapping period above (ramp rows ``t -> t+1`` of the
shard's last period, reference ``opf.py:468-479``) and one below when storage
SoC chains link ``t-1 -> t`` (``opf.py:585-597``).  The caller writes the
boundary variables into both shards, so cons / jac / hess need **no
per-set communication**; only the objective is a sum over ranks
(``torch.distributed.all_reduce``, NCCL over NVLink on the B200 box).

Each shard carries int64 maps to the global (unsharded) model -- variables,
rows, raw Jacobian slots, raw Hessian slots -- used to verify that the
reassembled shard results equal the global callbacks bit-for-bit, and to
scatter/gather x, y and outputs.  The maps come from the global record keys
(element * T + period) the builder attaches to every table.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ModelError
from .opf import _load_case, _OPFBuilder


def period_windows(T: int, n: int):
    """Contiguous, balanced partition of ``range(T)`` into ``n`` blocks."""
    if not 1 <= n <= T:
        raise ModelError(f"cannot split {T} periods into {n} shards")
    bounds = np.linspace(0, T, n + 1).round().astype(int)
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(n)]


@dataclass(eq=False)
class Shard:
    model: object
    window: tuple  # (c0, c1, v0, v1)
    var_map: np.ndarray | None = None  # shard var -> global var
    owned_vars: np.ndarray | None = None  # shard vars whose period is in [c0, c1)
    row_map: np.ndarray | None = None
    jac_map: np.ndarray | None = None
    hess_map: np.ndarray | None = None


def mpopf_shard(case, curve, rank: int, n_shards: int, corrective_action_ratio: float = 0.25,
                storage_complementarity_constraint: bool = False, form: str = "polar",
                lower_to_gpu: bool = True) -> Shard:
    """Rank ``rank``'s period shard of ``mpopf_model(case, curve, ...)``."""
    case = _load_case(case)
    curve = np.asarray(curve, dtype=np.float64)
    T = curve.size
    if T < 2:
        raise ModelError("period sharding needs a multi-period model")
    c0, c1 = period_windows(T, n_shards)[rank]
    has_storage = bool(case.storage)
    v0 = c0 - 1 if (has_storage and c0 > 0) else c0
    v1 = min(c1 + 1, T)
    pd0 = np.array([b.pd for b in case.buses])
    qd0 = np.array([b.qd for b in case.buses])
    builder = _OPFBuilder(case, form, np.outer(curve, pd0), np.outer(curve, qd0), corrective_action_ratio,
                          has_storage, storage_complementarity_constraint, None, window=(c0, c1, v0, v1))
    model = builder.build(lower_to_gpu)[0]
    return Shard(model=model, window=(c0, c1, v0, v1))


def attach_maps(shard: Shard, global_model) -> Shard:
    """Compute the shard -> global maps against the (host-only) global model."""
    c0, c1, v0, v1 = shard.window
    maps = attach_maps_generic(shard.model, global_model, np.arange(v0, v1), (c0, c1))
    shard.var_map, shard.owned_vars, shard.row_map, shard.jac_map, shard.hess_map = maps
    return shard


def attach_maps_generic(sm, gm, local_periods, owned=None):
    """Maps for a shard whose grid blocks hold the global periods/instances
    ``local_periods`` (in local order); ``owned = (c0, c1)`` marks the
    variables whose period the shard owns."""
    local_periods = np.asarray(local_periods, dtype=np.int64)
    var_map = np.empty(sm.nvar, dtype=np.int64)
    owned_mask = np.zeros(sm.nvar, dtype=bool)
    if len(sm.variables) != len(gm.variables):
        raise ModelError("shard and global models register different variable blocks")
    for sb, gb in zip(sm.variables, gm.variables):
        n = sb.shape[0]
        if len(gb.shape) == 1:  # static block: identical
            var_map[sb.offset:sb.offset + sb.size] = gb.offset + np.arange(gb.size)
            owned_mask[sb.offset:sb.offset + sb.size] = True
            continue
        T = gb.shape[1]
        Tv = sb.shape[1]
        if Tv != local_periods.size:
            raise ModelError("shard block period count does not match its period list")
        i = np.repeat(np.arange(n), Tv)
        t = np.tile(local_periods, n)
        var_map[sb.offset:sb.offset + sb.size] = gb.offset + i * T + t
        if owned is not None:
            owned_mask[sb.offset:sb.offset + sb.size] = (t >= owned[0]) & (t < owned[1])
    sp, gp = sm.plan, gm.plan
    if len(sp.obj_terms) != len(gp.obj_terms) or len(sp.con_terms) != len(gp.con_terms):
        raise ModelError("shard and global models register different term blocks")

    def rec_map(stp, gtp):
        gk = getattr(gtp.table, "_rkey", None)
        sk = getattr(stp.table, "_rkey", None)
        if gk is None or sk is None:
            raise ModelError("tables lack record keys; build both models with the OPF builders")
        at = np.searchsorted(gk, sk)
        if at.size and (at.max() >= gk.size or not np.array_equal(gk[at], sk)):
            raise ModelError("shard records not found in the global model")
        return at

    row_map = np.empty(sm.ncon, dtype=np.int64)
    jac_map = np.empty(sp.n_jac_slots, dtype=np.int64)
    hess_map = np.empty(sp.n_hess_slots, dtype=np.int64)
    for stp, gtp in zip(sp.obj_terms + sp.con_terms, gp.obj_terms + gp.con_terms):
        R = rec_map(stp, gtp)
        if stp.kind == "constraint":
            row_map[stp.row_offset:stp.row_offset + stp.nrec] = gtp.row_offset + R
        if stp.kind != "objective":
            for s in range(stp.tape.k):
                lo = stp.jac_slices[s][0]
                jac_map[lo:lo + stp.nrec] = gtp.jac_slices[s][0] + R
        for sp_pair, gp_pair in zip(stp.hess_pairs, gtp.hess_pairs):
            hess_map[sp_pair.start:sp_pair.start + stp.nrec] = gp_pair.start + R
    return var_map, owned_mask, row_map, jac_map, hess_map
