"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tools/make_goldens.py

It imports the reference package read-only from /root/reference/pkg/src,
builds each fixture model with the reference builders, evaluates the five
callbacks (plus compressed J/H) at seeded points and writes
``tests/golden/<name>.npz``.  Case data is stored as per-unit arrays so the
fixture can be rebuilt on a machine without the reference (the GPU box).
The fixtures pin both the oracle (``oracle/``) and the CUDA path.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_DATA = Path("/root/reference/pkg/data")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import simdnlp as ref  # noqa: E402
from simdnlp import autodiff as rad  # noqa: E402
from simdnlp.derivcheck import random_interior_point  # noqa: E402

from paper_2510_12897_b200 import synth  # noqa: E402
from paper_2510_12897_b200.casearrays import case_to_arrays  # noqa: E402


def ref_case_from_ours(c):
    from simdnlp import matpower as m

    return m.CaseData(
        c.name, c.base_mva,
        [m.Bus(b.bus_id, b.bus_type, b.pd, b.qd, b.gs, b.bs, b.vmax, b.vmin) for b in c.buses],
        [m.Gen(g.bus_id, g.pmin, g.pmax, g.qmin, g.qmax, g.status, g.c2, g.c1, g.c0) for g in c.gens],
        [m.Branch(b.f_bus, b.t_bus, b.r, b.x, b.b_charging, b.rate_a, b.tap, b.shift, b.status,
                  b.angmin, b.angmax) for b in c.branches],
        [m.Storage(s.bus_id, s.energy_rating, s.charge_rating, s.discharge_rating, s.eta_charge,
                   s.eta_discharge) for s in c.storage],
    )


def our_case_from_ref(c):
    from paper_2510_12897_b200 import matpower as m

    return m.CaseData(
        c.name, c.base_mva,
        [m.Bus(b.bus_id, b.bus_type, b.pd, b.qd, b.gs, b.bs, b.vmax, b.vmin) for b in c.buses],
        [m.Gen(g.bus_id, g.pmin, g.pmax, g.qmin, g.qmax, g.status, g.c2, g.c1, g.c0) for g in c.gens],
        [m.Branch(b.f_bus, b.t_bus, b.r, b.x, b.b_charging, b.rate_a, b.tap, b.shift, b.status,
                  b.angmin, b.angmax) for b in c.branches],
        [m.Storage(s.bus_id, s.energy_rating, s.charge_rating, s.discharge_rating, s.eta_charge,
                   s.eta_discharge) for s in c.storage],
    )


def custom_models():
    """Small non-OPF models mirroring reference test_autodiff fixtures."""
    from simdnlp import DataTable, ModelCore, cos, exp, field, log, sin, sqrt

    out = {}
    core = ModelCore()
    x = core.add_variable(2)
    core.add_objective(x["a"] * x["b"], DataTable({"a": np.array([0]), "b": np.array([1])}))
    out["product"] = core.compile()

    core = ModelCore()
    x = core.add_variable(3)
    core.add_objective(x["a"] * x["b"] + x["a"] ** 3,
                       DataTable({"a": np.array([0, 1, 2]), "b": np.array([0, 2, 2])}))
    out["dupvar"] = core.compile()

    core = ModelCore()
    x = core.add_variable(2, lower=[0.2, 0.3], upper=[3.0, 3.0], start=1.0)
    t = DataTable({"i": np.array([0, 1, 0]), "j": np.array([1, 0, 1]), "w": np.array([0.7, 1.3, 2.1])})
    kern = (sin(x["i"]) + cos(x["j"]) * exp(x["i"]) - log(x["j"]) / sqrt(x["i"])
            + x["i"] ** 3 - (-x["j"]) + field("w") ** x["i"] + x["i"] / x["j"])
    core.add_objective(kern, t)
    core.add_constraint(kern * x["j"] - 2.0 * x["i"] ** -2, t)
    out["allops"] = core.compile()

    core = ModelCore()
    x = core.add_variable(4, lower=0.1, upper=2.0, start=1.0)
    base = core.add_constraint(x["i"] ** 2 - field("c"), DataTable({"i": np.array([0, 1, 2]), "c": np.array([1.0, 2.0, 3.0])}))
    core.modify_constraint(base, 2.0 * x["k"] * x["i"], DataTable(
        {"k": np.array([3, 3, 0, 1]), "i": np.array([0, 1, 1, 2]), "row": np.array([0, 1, 1, 2])}))
    core.modify_constraint(base, -x["k"], DataTable({"k": np.array([2, 2]), "row": np.array([2, 0])}))
    core.add_constraint(x["i"] * 0.0 + x["k"] - x["k"], DataTable({"i": np.array([0, 1]), "k": np.array([2, 3])}))
    core.add_objective(x["a"] ** x["b"], DataTable({"a": np.array([0, 1]), "b": np.array([1, 2])}))
    out["augments"] = core.compile()
    return out


def fixtures():
    fx = []
    for name in ("case3", "case5", "case14"):
        case = ref.parse_case_file(REF_DATA / f"{name}.m")
        for form in ("polar", "rect"):
            fx.append((f"{name}_{form}", dict(kind="opf", form=form), case,
                       lambda c=case, f=form: ref.opf_model(c, form=f)[0]))
    strg = ref.parse_case_file(REF_DATA / "case5_strg.m")
    curve = np.array([1.0, 0.9, 1.1, 0.95])
    fx.append(("case5_strg_mp4_polar", dict(kind="mpopf", form="polar", curve=curve.tolist(),
                                           car=0.25, complementarity=True), strg,
               lambda: ref.mpopf_model(strg, curve, 0.25, True, form="polar")[0]))
    fx.append(("case5_strg_mp4_rect", dict(kind="mpopf", form="rect", curve=curve.tolist(),
                                          car=0.25, complementarity=False), strg,
               lambda: ref.mpopf_model(strg, curve, 0.25, False, form="rect")[0]))
    syn = ref_case_from_ours(synth.synthetic_case(60, 12, 90, seed=7, name="syn60"))
    fx.append(("syn60_polar", dict(kind="opf", form="polar"), syn,
               lambda: ref.opf_model(syn, form="polar")[0]))
    syn_mp = ref_case_from_ours(synth.synthetic_case(30, 6, 45, seed=3, name="syn30"))
    curve6 = synth.demand_curve(6)
    fx.append(("syn30_mp6_polar", dict(kind="mpopf", form="polar", curve=curve6.tolist(), car=0.25,
                                      complementarity=False), syn_mp,
               lambda: ref.mpopf_model(syn_mp, curve6, 0.25, form="polar")[0]))
    fx.append(("lv10", dict(kind="lv", n=10), None, lambda: ref.luksan_vlcek_model(10)[0]))
    for nm, mdl in custom_models().items():
        fx.append((nm, dict(kind="custom", which=nm), None, lambda m=mdl: m))
    return fx


def evaluate(model, x, y, w):
    g = np.empty(model.nvar)
    c = np.empty(model.ncon)
    J = np.empty(model.plan.n_jac_slots)
    H = np.empty(model.plan.n_hess_slots)
    f = rad.eval_objective(model, x)
    rad.eval_gradient(model, x, g)
    rad.eval_constraints(model, x, c)
    rad.eval_jacobian(model, x, J)
    rad.eval_hessian(model, x, y, w, H)
    return f, g, c, J, H


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    index = {}
    for name, spec, case, build in fixtures():
        model = build()
        jr, jc = rad.jacobian_structure(model)
        hr, hc = rad.hessian_structure(model)
        jp = rad.compress_coordinates(jr, jc)
        hp = rad.compress_coordinates(hr, hc)
        arrays = dict(
            nvar=model.nvar, ncon=model.ncon, lower=model.lower, upper=model.upper, start=model.start,
            con_lower=model.con_lower, con_upper=model.con_upper,
            jac_rows=jr, jac_cols=jc, hess_rows=hr, hess_cols=hc,
            jc_rows=jp.rows, jc_cols=jp.cols, jc_map=jp.slot_map,
            hc_rows=hp.rows, hc_cols=hp.cols, hc_map=hp.slot_map,
        )
        tapes = [tp.tape.instr for tp in model.plan.obj_terms + model.plan.con_terms]
        arrays["tapes_json"] = np.frombuffer(json.dumps(tapes).encode(), dtype=np.uint8)
        for p, seed in enumerate((0, 1)):
            rng = np.random.default_rng(seed)
            x = random_interior_point(model, rng)
            y = rng.uniform(-1.0, 1.0, size=model.ncon)
            w = 1.0 if p == 0 else -0.75
            f, g, c, J, H = evaluate(model, x, y, w)
            arrays.update({
                f"x{p}": x, f"y{p}": y, f"w{p}": w, f"obj{p}": f, f"grad{p}": g, f"cons{p}": c,
                f"jac{p}": J, f"hess{p}": H,
                f"jacc{p}": jp.sum_values(J), f"hessc{p}": hp.sum_values(H),
            })
        if case is not None:
            arrays.update({f"case_{k}": v for k, v in case_to_arrays(our_case_from_ref(case)).items()})
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        index[name] = spec
        print(f"{name:24s} nvar={model.nvar:6d} ncon={model.ncon:6d} "
              f"jac={model.plan.n_jac_slots:7d} hess={model.plan.n_hess_slots:7d}")
    (OUT / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
