"""End-to-end host-buffer throughput (exa_eval_set_host, pinned buffers, NS
streams in round robin) with and without host mirrors, interleaved A/B runs
on one box so that host noise hits both.

    python tools/e2e_timing.py [workload] [sets per run] [runs]
Prints one JSON line per run and a summary line (medians).
"""
import ctypes as C
import json
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 600
RUNS = int(sys.argv[3]) if len(sys.argv) > 3 else 5
NS = int(os.environ.get("EXA_E2E_STREAMS", "3"))
model = build_workload(name, lower_to_gpu=False)
plans = {}
for mir in ("1", "0"):
    os.environ["EXA_HOST_MIRROR"] = mir
    plans[mir] = DevicePlan(model, 0)
lib = _lib.load()
x, y, w = eval_inputs(model, 0)
n = (model.ncon, model.plan.n_jac_slots, model.plan.n_hess_slots)
slots = []
for k in range(NS):
    slots.append({"st": torch.cuda.Stream(), "x": torch.from_numpy(x).pin_memory(), "y": torch.from_numpy(y).pin_memory(),
                  "o": [torch.empty(m, dtype=torch.float64).pin_memory() for m in n], "ws": {}})
    for key, p in plans.items():
        ws = C.c_void_p()
        _lib.check(lib.exa_workspace_create(p.handle, C.byref(ws)), "ws")
        slots[-1]["ws"][key] = ws


def run(key, count, sync_each=False):
    p = plans[key]
    t0 = time.perf_counter()
    for i in range(count):
        sl = slots[i % NS]
        _lib.check(lib.exa_eval_set_host(p.handle, sl["ws"][key], sl["x"].data_ptr(), sl["y"].data_ptr(), w,
                                         *(t.data_ptr() for t in sl["o"]), C.c_void_p(sl["st"].cuda_stream)), "set_host")
        if sync_each:
            sl["st"].synchronize()
    for sl in slots:
        sl["st"].synchronize()
    return count / (time.perf_counter() - t0)


for key in plans:
    run(key, 3 * NS)
res = {"1": [], "0": []}
for r in range(RUNS):
    for key in ("1", "0") if r % 2 == 0 else ("0", "1"):
        v = run(key, N)
        res[key].append(v)
        print(json.dumps({"run": r, "mirrors": key, "sets_per_s": v}), flush=True)
lay = plans["1"].layout
mb = 8 * sum(int(m[:, 1].sum()) for m in (lay.mirror_jac, lay.mirror_hess) if len(m))
print(json.dumps({"workload": name, "streams": NS, "sets_per_run": N, "median_mirrors": statistics.median(res["1"]),
                  "median_no_mirrors": statistics.median(res["0"]), "mirrored_bytes": mb,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("EXA_")}}), flush=True)
