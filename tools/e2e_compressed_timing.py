"""End-to-end compressed host path (exa_eval_set_compressed_host, pinned
buffers, NS streams in round robin): direct Jacobian entries on / off
(EXA_JDIRECT read per plan), interleaved runs on one box.

    python tools/e2e_compressed_timing.py [workload] [sets per run] [runs]
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

from paper_2510_12897_b200 import _lib, model_patterns
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 400
RUNS = int(sys.argv[3]) if len(sys.argv) > 3 else 4
NS = 4
model = build_workload(name, lower_to_gpu=False)
jp, hp = model_patterns(model)
lib = _lib.load()
x, y, w = eval_inputs(model, 0)
var = {}
for jd in ("1", "0"):
    os.environ["EXA_JDIRECT"] = jd
    p = DevicePlan(model, 0)
    hj, hh = jp.device_handle(p, "jac"), hp.device_handle(p, "hess")
    slots = []
    for k in range(NS):
        ws = C.c_void_p()
        _lib.check(lib.exa_workspace_create(p.handle, C.byref(ws)), "ws")
        slots.append({"st": torch.cuda.Stream(), "ws": ws, "x": torch.from_numpy(x).pin_memory(),
                      "y": torch.from_numpy(y).pin_memory(),
                      "o": [torch.empty(m, dtype=torch.float64).pin_memory() for m in (model.ncon, jp.nnz, hp.nnz)]})
    var[jd] = (p, hj, hh, slots)


def run(jd, count):
    p, hj, hh, slots = var[jd]
    t0 = time.perf_counter()
    for i in range(count):
        sl = slots[i % NS]
        _lib.check(lib.exa_eval_set_compressed_host(p.handle, sl["ws"], hj, hh, sl["x"].data_ptr(), sl["y"].data_ptr(),
                                                    w, *(t.data_ptr() for t in sl["o"]),
                                                    C.c_void_p(sl["st"].cuda_stream)), "set_compressed_host")
    for sl in slots:
        sl["st"].synchronize()
    return count / (time.perf_counter() - t0)


for jd in var:
    run(jd, 3 * NS)
res = {"1": [], "0": []}
for r in range(RUNS):
    for jd in (("1", "0") if r % 2 == 0 else ("0", "1")):
        res[jd].append(run(jd, N))
a, b = var["1"][3][0]["o"], var["0"][3][0]["o"]
same = all(torch.equal(u.view(torch.int64), v.view(torch.int64)) for u, v in zip(a, b))
print(json.dumps({"workload": name, "median_direct": statistics.median(res["1"]), "median_no_direct": statistics.median(res["0"]),
                  "runs": res, "outputs_bit_equal": same}), flush=True)
