"""Batched N-1 security-constrained AC-OPF (BASELINE config 5).

The reference has no N-1 model (SPEC non-goal); SURVEY §8c composes it from
the reference API: instance 0 is the base case, instance k >= 1 is the case
with branch ``contingencies[k-1]`` out of service (``opf.py:205`` drops
inactive branches), and linking rows ``pg_k - pg_0`` (the F10 tape,
``opf.py:468-479``) tie every contingency's dispatch to the base case
(preventive security: ``lb = ub = 0``, or ``±ratio·(Pmax - Pmin)``).

SIMD layout: every family is ONE block over all (element, instance) records,
element-major like the multi-period model (``i * S + k``), so the whole batch
is ~16 generated kernels regardless of the number of contingencies.  The
variable layout is uniform over instances (an outaged branch keeps its p/q
variables, which simply appear in no row of that instance).

Sharding: rank s owns instances ``[c0, c1)`` and holds variables for
``{0} ∪ [c0, c1)`` -- the base-case generator outputs are the only linking
data (238 doubles at case2000), broadcast once per x update; cons/jac/hess
need no collective, the objective (base cost) lives on the rank owning 0.
"""

from __future__ import annotations

import time
from types import SimpleNamespace

import numpy as np

from .core import DataTable, ModelCore, ModelError
from .expressions import cos, field, sin
from .matpower import branch_admittance, validate_case
from .opf import _keyed, _load_case, _midpoint, angle_rows_eligible


def instance_windows(n_instances: int, n: int):
    from .sharding import period_windows

    return period_windows(n_instances, n)


def scopf_model(case, contingencies, form: str = "polar", corrective_ratio: float | None = None,
                owned=None, lower_to_gpu: bool = True):
    """Batched N-1 model.  ``owned = (c0, c1)`` builds the shard owning
    instances ``[c0, c1)`` (variables also for the base instance 0)."""
    t_start = time.perf_counter()
    case = _load_case(case)
    if form != "polar":
        raise ModelError("batched N-1 is provided for the polar formulation")
    errs = validate_case(case)
    if errs:
        raise ModelError("invalid case: " + "; ".join(errs))
    branches = [br for br in case.branches if br.status == 1]
    gens = [g for g in case.gens if g.status == 1]
    nbr, ng, nb = len(branches), len(gens), case.n_bus
    cont = np.asarray(contingencies, dtype=np.int64)
    if cont.size and (cont.min() < 0 or cont.max() >= nbr):
        raise ModelError("contingency index outside the active branch list")
    S = cont.size + 1
    c0, c1 = owned if owned is not None else (0, S)
    own = np.arange(c0, c1, dtype=np.int64)
    local = own if c0 == 0 else np.concatenate([[0], own]).astype(np.int64)
    Sl = local.size
    lpos = np.full(S, -1, dtype=np.int64)
    lpos[local] = np.arange(Sl)
    out_branch = np.full(S, -1, dtype=np.int64)
    out_branch[1:] = cont

    pos = case.bus_index()
    ref = next(i for i, b in enumerate(case.buses) if b.bus_type == 3)
    adm = [branch_admittance(br) for br in branches]
    fpos = np.array([pos[br.f_bus] for br in branches], dtype=np.int64)
    tpos = np.array([pos[br.t_bus] for br in branches], dtype=np.int64)
    gpos = np.array([pos[g.bus_id] for g in gens], dtype=np.int64)

    def flat(i, k):
        return np.asarray(i, dtype=np.int64) * Sl + lpos[np.asarray(k, dtype=np.int64)]

    def vtile(values):
        return np.repeat(np.asarray(values, dtype=np.float64), Sl)

    def records(n, active=None):
        """(element, instance) over owned instances, element-major; ``active``
        (n x S bool) filters records (outaged branches)."""
        rep = np.repeat(np.arange(n, dtype=np.int64), own.size)
        k = np.tile(own, n)
        if active is not None:
            keep = active[rep, k]
            rep, k = rep[keep], k[keep]
        return rep, k

    core = ModelCore()
    v = SimpleNamespace()
    c = SimpleNamespace()
    vmax = np.array([b.vmax for b in case.buses])
    vmin = np.array([b.vmin for b in case.buses])
    v.va = core.add_variable((nb, Sl), start=0.0, name="va")
    v.vm = core.add_variable((nb, Sl), lower=vtile(vmin), upper=vtile(vmax), start=1.0, name="vm")
    pg_lo, pg_hi = vtile([g.pmin for g in gens]), vtile([g.pmax for g in gens])
    qg_lo, qg_hi = vtile([g.qmin for g in gens]), vtile([g.qmax for g in gens])
    v.pg = core.add_variable((ng, Sl), lower=pg_lo, upper=pg_hi, start=_midpoint(pg_lo, pg_hi), name="pg")
    v.qg = core.add_variable((ng, Sl), lower=qg_lo, upper=qg_hi, start=_midpoint(qg_lo, qg_hi), name="qg")
    v.p = core.add_variable((2 * nbr, Sl), start=0.0, name="p")
    v.q = core.add_variable((2 * nbr, Sl), start=0.0, name="q")

    # base-case generation cost (instance 0 only)
    g_rep = np.arange(ng, dtype=np.int64) if c0 == 0 else np.zeros(0, dtype=np.int64)
    g_k = np.zeros(g_rep.size, dtype=np.int64)
    mw = v.pg["g"] * case.base_mva
    core.add_objective(
        field("c2") * mw**2 + field("c1") * mw + field("c0"),
        _keyed(DataTable({"g": flat(g_rep, g_k),
                          "c2": np.array([g.c2 for g in gens])[g_rep],
                          "c1": np.array([g.c1 for g in gens])[g_rep],
                          "c0": np.array([g.c0 for g in gens])[g_rep]}), g_rep, g_k, S))
    c.c_ref_angle = core.add_constraint(
        v.va["i"], _keyed(DataTable({"i": flat(np.full(own.size, ref), own)}),
                          np.zeros(own.size, dtype=np.int64), own, S))

    active = np.ones((nbr, S), dtype=bool)
    active[out_branch[1:], np.arange(1, S)] = False
    rep, k = records(nbr, active)
    g_s = np.array([a.g for a in adm])
    b_s = np.array([a.b for a in adm])
    tr = np.array([a.tr for a in adm])
    ti = np.array([a.ti for a in adm])
    tm = np.array([a.tm for a in adm])
    b_fr = np.array([a.b_fr for a in adm])
    b_to = np.array([a.b_to for a in adm])
    g_fr = np.array([a.g_fr for a in adm])
    g_to = np.array([a.g_to for a in adm])
    from_dir = np.arange(nbr, dtype=np.int64)
    to_dir = nbr + from_dir

    def flow_kernel(flow):
        delta = v.va["i"] - v.va["j"]
        return (field("a1") * v.vm["i"] ** 2
                + v.vm["i"] * v.vm["j"] * (field("a2") * cos(delta) + field("a3") * sin(delta))
                - flow["d"])

    def table(side, other, a1, a2, a3, direction):
        return _keyed(DataTable({"i": flat(side[rep], k), "j": flat(other[rep], k), "d": flat(direction[rep], k),
                                 "a1": a1[rep], "a2": a2[rep], "a3": a3[rep]}), rep, k, S)

    c.c_from_active_power_flow = core.add_constraint(flow_kernel(v.p), table(
        fpos, tpos, (g_s + g_fr) / tm, (-g_s * tr + b_s * ti) / tm, (-b_s * tr - g_s * ti) / tm, from_dir))
    c.c_from_reactive_power_flow = core.add_constraint(flow_kernel(v.q), table(
        fpos, tpos, -(b_s + b_fr) / tm, (b_s * tr + g_s * ti) / tm, (-g_s * tr + b_s * ti) / tm, from_dir))
    c.c_to_active_power_flow = core.add_constraint(flow_kernel(v.p), table(
        tpos, fpos, g_s + g_to, (-g_s * tr - b_s * ti) / tm, (-b_s * tr + g_s * ti) / tm, to_dir))
    c.c_to_reactive_power_flow = core.add_constraint(flow_kernel(v.q), table(
        tpos, fpos, -(b_s + b_to), (b_s * tr - g_s * ti) / tm, (-g_s * tr - b_s * ti) / tm, to_dir))

    # balances (all buses, owned instances) and device augments
    bus_rep, bus_k = records(nb)
    gs = np.array([b.gs for b in case.buses])
    bs = np.array([b.bs for b in case.buses])
    v2 = v.vm["b"] ** 2
    pdv = np.array([b.pd for b in case.buses])
    qdv = np.array([b.qd for b in case.buses])
    p_kernel, p_cols = -field("pd"), {"pd": pdv[bus_rep]}
    if np.any(gs != 0.0):
        p_kernel = p_kernel - field("gs") * v2
        p_cols.update(gs=gs[bus_rep], b=flat(bus_rep, bus_k))
    q_kernel, q_cols = -field("qd"), {"qd": qdv[bus_rep]}
    if np.any(bs != 0.0):
        q_kernel = q_kernel + field("bs") * v2
        q_cols.update(bs=bs[bus_rep], b=flat(bus_rep, bus_k))
    p_bal = core.add_constraint(p_kernel, _keyed(DataTable(p_cols), bus_rep, bus_k, S))
    q_bal = core.add_constraint(q_kernel, _keyed(DataTable(q_cols), bus_rep, bus_k, S))
    c.c_active_power_balance, c.c_reactive_power_balance = p_bal, q_bal
    own_pos = np.full(S, -1, dtype=np.int64)
    own_pos[own] = np.arange(own.size)

    def bal_row(block, bus, kk):
        return block.row_offset + bus * own.size + own_pos[kk]

    gr, gk = records(ng)
    core.modify_constraint(p_bal, v.pg["g"], _keyed(DataTable(
        {"g": flat(gr, gk), "row": bal_row(p_bal, gpos[gr], gk)}), gr, gk, S))
    core.modify_constraint(q_bal, v.qg["g"], _keyed(DataTable(
        {"g": flat(gr, gk), "row": bal_row(q_bal, gpos[gr], gk)}), gr, gk, S))
    dir_active = np.concatenate([active, active])
    dr, dk = records(2 * nbr, dir_active)
    d_bus = np.concatenate([fpos, tpos])
    core.modify_constraint(p_bal, -v.p["d"], _keyed(DataTable(
        {"d": flat(dr, dk), "row": bal_row(p_bal, d_bus[dr], dk)}), dr, dk, S))
    core.modify_constraint(q_bal, -v.q["d"], _keyed(DataTable(
        {"d": flat(dr, dk), "row": bal_row(q_bal, d_bus[dr], dk)}), dr, dk, S))

    rate = np.array([br.rate_a for br in branches])
    lim_active = active & (rate > 0.0)[:, None]
    lr, lk = records(nbr, lim_active)
    thermal = v.p["d"] ** 2 + v.q["d"] ** 2
    ub = (rate**2)[lr]
    c.c_thermal_from = core.add_constraint(
        thermal, _keyed(DataTable({"d": flat(from_dir[lr], lk)}), lr, lk, S), lb=-np.inf, ub=ub)
    c.c_thermal_to = core.add_constraint(
        thermal, _keyed(DataTable({"d": flat(to_dir[lr], lk)}), lr, lk, S), lb=-np.inf, ub=ub)
    ang_ok = np.array([angle_rows_eligible(br) for br in branches], dtype=bool)
    ar, ak = records(nbr, active & ang_ok[:, None])
    c.c_angle_diff = core.add_constraint(
        v.va["i"] - v.va["j"],
        _keyed(DataTable({"i": flat(fpos[ar], ak), "j": flat(tpos[ar], ak)}), ar, ak, S),
        lb=np.array([branches[i].angmin for i in ar]), ub=np.array([branches[i].angmax for i in ar]))

    # linking: pg_k - pg_0 for every owned contingency instance
    lk_inst = own[own >= 1]
    li = np.repeat(np.arange(ng, dtype=np.int64), lk_inst.size)
    lkk = np.tile(lk_inst, ng)
    span = np.array([g.pmax - g.pmin for g in gens])[li]
    lim = 0.0 * span if corrective_ratio is None else corrective_ratio * span
    c.c_security = core.add_constraint(
        v.pg["i1"] - v.pg["i0"],
        _keyed(DataTable({"i0": flat(li, np.zeros(li.size, dtype=np.int64)), "i1": flat(li, lkk)}), li, lkk, S),
        lb=-lim, ub=lim)
    model = core.compile(lower_to_gpu=False)
    # element-major (element, instance) layout: variable (i, k) at i * Sl + k;
    # the device layout dispatches the set kernel's CTAs by instance window
    model.plan.batch_period = Sl
    if lower_to_gpu:
        model.to_device()
    model.build_seconds = time.perf_counter() - t_start
    model.instances = local
    return model, v, c


def scopf_shard(case, contingencies, rank: int, n_shards: int, **kw):
    S = len(contingencies) + 1
    c0, c1 = instance_windows(S, n_shards)[rank]
    model = scopf_model(case, contingencies, owned=(c0, c1), **kw)[0]
    return model, (c0, c1)


def attach_instance_maps(shard_model, global_model, owned):
    """Shard -> global maps (vars, owned-var mask, rows, J slots, H slots)."""
    from .sharding import attach_maps_generic

    return attach_maps_generic(shard_model, global_model, shard_model.instances, owned)
