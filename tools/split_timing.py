"""Concurrency experiment: heavy and light kernels on two free-running streams."""
import ctypes as C, json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["EXA_SPLIT"] = "1"
import numpy as np, torch
from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs, model_summary

model = build_workload("case13659", lower_to_gpu=False)
bps = model_summary(model)["bytes_per_set"]
R = 11
dev = torch.device("cuda", 0)
plans = [DevicePlan(model, 0) for _ in range(R)]
lib = _lib.load()
bufs = []
for r in range(R):
    x, y, w = eval_inputs(model, r)
    bufs.append([torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev),
                 torch.empty(model.ncon, dtype=torch.float64, device=dev),
                 torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev),
                 torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev)])
ws = []
for p in plans:
    h = C.c_void_p()
    _lib.check(lib.exa_workspace_create(p.handle, C.byref(h)))
    ws.append(h)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
S = 64


def run(mode):
    # mode "fork": normal exa_eval_set on s1 (fork/join inside); "graph": same captured
    for i in range(S * R):
        b = bufs[i % R]
        rc = lib.exa_eval_set(plans[i % R].handle, ws[i % R], b[0].data_ptr(), b[1].data_ptr(), 1.0,
                              b[2].data_ptr(), b[3].data_ptr(), b[4].data_ptr(), C.c_void_p(s1.cuda_stream))
        assert rc == 0


out = {}
for mode in ("eager",):
    run(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    run(mode)
    e1.record(s1)
    torch.cuda.synchronize()
    out[mode] = e0.elapsed_time(e1) * 1e3 / (S * R)
# graph capture of the same
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s1):
    run("graph")
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s1)
for _ in range(3):
    g.replay()
e1.record(s1)
torch.cuda.synchronize()
out["graph"] = e0.elapsed_time(e1) * 1e3 / (3 * S * R)
print(json.dumps(out))
