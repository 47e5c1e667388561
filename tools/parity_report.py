#!/usr/bin/env python
"""Per-config parity report of the CUDA callbacks (SURVEY §8c comparator).

    python tools/parity_report.py [--out gpurun_out/parity.json] [config ...]

For every BASELINE config (default: case14, case1354, case13659,
mp96_case1354, scen96_case1354, n1_case2000 at 1024 contingencies) at the
bench evaluation point (seed 0): the fused set kernel's c / J / H, the
separate cons / jac / hess kernels, the objective and the gradient, against

* the numpy oracle (the reference's arithmetic: pinned bit-exact to goldens
  the reference itself produced, tests/test_oracle_pinned.py), and
* the same oracle with correctly-rounded sin/cos (oracle/crtrig).

Recorded per array and per family: strict 1e-12 violations, IEEE-unequal
elements, zero-sign mismatches, max relative deviation, the
conditioning-scaled max (oracle/parity.py), and whether every violation
equals the CR oracle.  Runs on a B200 (the callbacks have no CPU path).
The zero-sign mode of the generated kernels is reported (EXA_EXACT_ZERO_SIGN).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CONFIGS = ("case14", "case1354", "case13659", "mp96_case1354", "scen96_case1354", "n1_case2000")


def run_config(name):
    import numpy as np
    import torch

    from oracle import crtrig
    from oracle import parity as P
    from oracle import tape_oracle as O
    from paper_2510_12897_b200 import autodiff as A
    from paper_2510_12897_b200.codegen import _DERIV_ZERO_ELISION
    from paper_2510_12897_b200.workloads import build_workload, eval_inputs

    t0 = time.perf_counter()
    model = build_workload(name, lower_to_gpu=True)
    x, y, w = eval_inputs(model, 0)
    plan = model.plan
    dev = torch.device("cuda", 0)
    xt, yt = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)

    def dev_out(n):
        return torch.full((n,), float("nan"), dtype=torch.float64, device=dev)

    c, J, H = dev_out(model.ncon), dev_out(plan.n_jac_slots), dev_out(plan.n_hess_slots)
    A.eval_callback_set(model, xt, yt, w, c, J, H)
    c2, J2, H2 = dev_out(model.ncon), dev_out(plan.n_jac_slots), dev_out(plan.n_hess_slots)
    A.eval_constraints(model, xt, c2)
    A.eval_jacobian(model, xt, J2)
    A.eval_hessian(model, xt, yt, w, H2)
    g = dev_out(model.nvar)
    A.eval_gradient(model, xt, g)
    f = A.eval_objective(model, xt)
    torch.cuda.synchronize(dev)
    got = tuple(t.cpu().numpy() for t in (c, J, H))
    sep = tuple(t.cpu().numpy() for t in (c2, J2, H2))
    g = g.cpu().numpy()
    del c, J, H, c2, J2, H2
    torch.cuda.empty_cache()
    t_gpu = time.perf_counter() - t0

    t1 = time.perf_counter()
    ref = O.eval_set(plan, x, y, w)
    f_ref = O.eval_objective(plan, x)
    g_ref = np.empty(model.nvar)
    O.eval_gradient(plan, x, g_ref)
    O.use_trig(crtrig.TRIG)
    try:
        cr = O.eval_set(plan, x, y, w)
        f_cr = O.eval_objective(plan, x)
        g_cr = np.empty(model.nvar)
        O.eval_gradient(plan, x, g_cr)
    finally:
        O.use_trig(None)
    t_oracle = time.perf_counter() - t1

    rep = P.report(plan, x, y, w, got, ref, cr)
    rep["arrays"]["obj"] = P.scalar_stats(f, f_ref, f_cr)
    rep["arrays"]["grad"] = P.scalar_stats(g, g_ref, g_cr)
    rep["separate_callbacks_bit_equal_set"] = {
        k: P.bit_equal(a, b) for k, a, b in zip(("cons", "jac", "hess"), got, sep)}
    rep["bit_equal_cr_oracle"] = {k: P.bit_equal(a, b) for k, a, b in zip(("cons", "jac", "hess"), got, cr)}
    rep["bit_equal_cr_oracle"]["grad"] = P.bit_equal(g, g_cr)
    rep["bit_equal_cr_oracle"]["obj"] = P.bit_equal(np.array([f]), np.array([f_cr]))
    rep["ieee_equal_cr_oracle"] = {k: P.ieee_equal(a, b) for k, a, b in zip(("cons", "jac", "hess"), got, cr)}
    rep.update(config=name, nvar=model.nvar, ncon=model.ncon, jac_slots=plan.n_jac_slots,
               hess_slots=plan.n_hess_slots, eval_point="workloads.eval_inputs(model, seed=0)",
               zero_sign_mode="relaxed (+0.0 structural zeros)" if _DERIV_ZERO_ELISION else "exact",
               seconds={"gpu": round(t_gpu, 2), "oracles": round(t_oracle, 2)})
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=list(CONFIGS))
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "parity.json"))
    ap.add_argument("--no-families", action="store_true")
    args = ap.parse_args()
    out = {"tool": "tools/parity_report.py", "rtol": 1e-12,
           "exact_zero_sign_env": os.environ.get("EXA_EXACT_ZERO_SIGN", "0"), "configs": {}}
    for name in args.configs:
        rep = run_config(name)
        if args.no_families:
            rep.pop("families", None)
        out["configs"][name] = rep
        a = rep["arrays"]
        print(json.dumps({"config": name, **{k: (v["strict_violations"], v["ieee_unequal"], v["zero_sign_mismatch"],
                                                 v.get("cr_oracle_unequal"))
                                             for k, v in a.items()}}), flush=True)
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
