"""Benchmark workloads (BASELINE.json configs) and their algorithmic bytes.

Configs:

* ``case14``      bundled-style small case (parity; CPU-runnable reference);
* ``case1354``    pglib case1354_pegase-shaped, polar, static;
* ``case13659``   pglib case13659_pegase-shaped, polar, static (headline);
* ``mp96_case1354``  96-period MPOPF with ramping on the 1354-shaped network;
* ``n1_case2000``    N-1 batch on the case2000-shaped network (see :mod:`.scopf`);
* ``scen96_case1354`` 96 independent load scenarios of the 1354-shaped network
  (north_star "load scenarios": the multi-period builder without ramp rows,
  ``corrective_action_ratio=None``, scenario load factors U(0.8, 1.2)).

``algorithmic_bytes`` is SURVEY §8(d)'s compulsory-traffic count for one
callback set (cons + jac + hess): x and y once, every term parameter once
(fp64 fields, int32 index columns, +1 int32 row column for augments) as the
device layout stores it -- per record, or once per element for the periodic
columns of element-major batched models (MP96: 43.2 -> 6.0 MB) -- every
output once.  COO structure arrays are not re-read per set.
"""

from __future__ import annotations

import numpy as np

from .opf import mpopf_model, opf_model
from .synth import demand_curve, pglib_shaped

WORKLOADS = ("case14", "case1354", "case2000", "case13659", "mp96_case1354", "n1_case2000", "scen96_case1354")
SHARDED = ("mp", "n1", "scen")  # batched configs: one instance sharded over the ranks


def scenario_factors(S: int, seed: int = 7):
    return np.random.default_rng(seed).uniform(0.8, 1.2, S)


def _parse(name: str):
    head, base = name.split("_", 1)
    return head, base


def n1_contingencies(case, K: int):
    """Branches 0..K-1 outaged one at a time."""
    return list(range(min(K, len([b for b in case.branches if b.status == 1]))))


def build_workload(name: str, lower_to_gpu: bool = True, seed: int = 1, rank: int = 0, world: int = 1):
    """Model for a benchmark config; batched configs return rank's shard."""
    if name in ("case14", "case1354", "case2000", "case13659"):
        case = pglib_shaped(name, seed=seed)
        return opf_model(case, form="polar", lower_to_gpu=lower_to_gpu)[0]
    head, base = _parse(name)
    case = pglib_shaped(base, seed=seed)
    if head.startswith("mp"):
        T = int(head[2:])
        if world == 1:
            return mpopf_model(case, demand_curve(T), corrective_action_ratio=0.25, form="polar",
                               lower_to_gpu=lower_to_gpu)[0]
        from .sharding import mpopf_shard

        return mpopf_shard(case, demand_curve(T), rank, world, 0.25, lower_to_gpu=lower_to_gpu).model
    if head.startswith("scen"):
        S = int(head[4:])
        if world == 1:
            return mpopf_model(case, scenario_factors(S), corrective_action_ratio=None, form="polar",
                               lower_to_gpu=lower_to_gpu)[0]
        from .sharding import mpopf_shard

        return mpopf_shard(case, scenario_factors(S), rank, world, None, lower_to_gpu=lower_to_gpu).model
    if head.startswith("n1"):
        K = int(head[2:]) if len(head) > 2 else 1024
        from .scopf import instance_windows, scopf_model

        cont = n1_contingencies(case, K)
        owned = instance_windows(len(cont) + 1, world)[rank] if world > 1 else None
        return scopf_model(case, cont, owned=owned, lower_to_gpu=lower_to_gpu)[0]
    raise KeyError(name)


def _term_param_bytes(tp, period) -> int:
    """Parameter bytes of one term as the device layout stores them: fp64
    fields and int32 index columns per record (+ the augment row column),
    except periodic columns of element-major batched models, stored once per
    element (``device._periodic``: MP models' branch admittances, costs,
    limits and (bus, period) variable positions)."""
    from .device import _periodic

    red = _periodic(tp, period) or {"fcols": {}, "icols": {}}
    n = tp.nrec
    b = sum(8 * (red["fcols"][fi].size if fi in red["fcols"] else n) for fi in range(len(tp.tape.field_names)))
    b += sum(4 * (red["icols"][c].size if c in red["icols"] else n) for c in range(len(tp.tape.index_names)))
    return b + (4 * n if tp.kind == "augment" else 0)


def _layout_period(plan):
    from .device import META_CONST_MAX_TERMS, PERIODIC

    specialised = len(plan.obj_terms) + len(plan.con_terms) <= META_CONST_MAX_TERMS
    return getattr(plan, "batch_period", None) if (PERIODIC and specialised) else None


def algorithmic_bytes(model) -> dict:
    plan = model.plan
    period = _layout_period(plan)
    params = sum(_term_param_bytes(tp, period) for tp in plan.obj_terms + plan.con_terms)
    parts = {
        "x": 8 * model.nvar,
        "y": 8 * model.ncon,
        "params": params,
        "cons": 8 * model.ncon,
        "jac": 8 * plan.n_jac_slots,
        "hess": 8 * plan.n_hess_slots,
    }
    parts["total"] = sum(parts.values())
    return parts


def algorithmic_bytes_mode(model, mode: str) -> int:
    """Compulsory bytes of ONE callback (``set``, ``cons``, ``jac``, ``hess``):
    x once, the multipliers for the Hessian, the parameters of the terms the
    callback evaluates (cons: every constraint-side term; jac: those with
    variables; hess: every term with variables, objective included), and
    the callback's own output."""
    if mode == "set":
        return algorithmic_bytes(model)["total"]
    plan = model.plan

    period = _layout_period(plan)

    def params(terms):
        return sum(_term_param_bytes(tp, period) for tp in terms)

    b = 8 * model.nvar
    if mode == "cons":
        return b + params(plan.con_terms) + 8 * model.ncon
    if mode == "jac":
        return b + params([tp for tp in plan.con_terms if tp.tape.k]) + 8 * plan.n_jac_slots
    if mode == "hess":
        return (b + 8 * model.ncon + params([tp for tp in plan.obj_terms + plan.con_terms if tp.tape.k])
                + 8 * plan.n_hess_slots)
    raise ValueError(mode)


def bench_models_for_precompile():
    """Host plans whose kernel modules build() pre-compiles (no GPU needed)."""
    out = []
    for name in ("case13659", "mp96_case1354"):
        out.append(build_workload(name, lower_to_gpu=False).plan)
    return out


def model_summary(model) -> dict:
    b = algorithmic_bytes(model)
    return {
        "nvar": model.nvar, "ncon": model.ncon,
        "jac_slots": model.plan.n_jac_slots, "hess_slots": model.plan.n_hess_slots,
        "bytes_per_set": b["total"], "bytes": b,
    }


def eval_inputs(model, seed: int = 0):
    from .synth import evaluation_point

    x, y, w = evaluation_point(model, seed)
    return np.ascontiguousarray(x), np.ascontiguousarray(y), w
