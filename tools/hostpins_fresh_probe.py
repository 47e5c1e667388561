"""A solver's pattern through the numpy set: outputs reused, x / y new arrays
every call.  Splits the time into the input copies and the call, for outputs
pageable (staged), locked in place, and page-locked (empty_pinned)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2510_12897_b200 import autodiff, empty_pinned, eval_callback_set  # noqa: E402
from paper_2510_12897_b200.workloads import build_workload, eval_inputs  # noqa: E402

m = build_workload(sys.argv[1] if len(sys.argv) > 1 else "case13659")
x, y, w = eval_inputs(m, 0)
nj, nh = m.plan.n_jac_slots, m.plan.n_hess_slots


def run(label, outs, fresh, n=60):
    for _ in range(3):
        xs, ys = (x.copy(), y.copy()) if fresh == "copy" else (x, y)
        eval_callback_set(m, xs, ys, w, *outs)
    tc = tcall = 0.0
    for _ in range(n):
        t0 = time.perf_counter()
        if fresh == "copy":
            xs, ys = x.copy(), y.copy()
        elif fresh == "pinned":
            xs, ys = empty_pinned(m.nvar), empty_pinned(m.ncon)
            xs[:], ys[:] = x, y
        else:
            xs, ys = x, y
        t1 = time.perf_counter()
        eval_callback_set(m, xs, ys, w, *outs)
        t2 = time.perf_counter()
        tc += t1 - t0
        tcall += t2 - t1
    print(f"{label:48s} inputs {1e6 * tc / n:6.0f} us  call {1e6 * tcall / n:6.0f} us", flush=True)


for fresh in ("same", "copy"):
    autodiff._PINS.enabled = False
    run(f"x/y {fresh}, outputs pageable (staged)", (np.empty(m.ncon), np.empty(nj), np.empty(nh)), fresh)
    autodiff._PINS.enabled = True
    run(f"x/y {fresh}, outputs locked in place", (np.empty(m.ncon), np.empty(nj), np.empty(nh)), fresh)
    autodiff._PINS.enabled = False
    run(f"x/y {fresh}, outputs empty_pinned", (empty_pinned(m.ncon), empty_pinned(nj), empty_pinned(nh)), fresh)
