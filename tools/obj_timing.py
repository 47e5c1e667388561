"""Objective / gradient callback timing (exa_eval_obj / exa_eval_grad),
graph of rotating replicas; EXA_NCU=1: a few eager calls for ncu.

    python tools/obj_timing.py case13659
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
model = build_workload(name, lower_to_gpu=False)
R = 4
dev = torch.device("cuda", 0)
plans = [DevicePlan(model, 0) for _ in range(R)]
lib = _lib.load()
xs = [torch.from_numpy(eval_inputs(model, r)[0]).to(dev) for r in range(R)]
f = torch.empty(R, dtype=torch.float64, device=dev)
g = [torch.empty(model.nvar, dtype=torch.float64, device=dev) for _ in range(R)]
st = torch.cuda.Stream(dev)
sh = C.c_void_p(st.cuda_stream)


def obj(i):
    assert lib.exa_eval_obj(plans[i % R].handle, None, xs[i % R].data_ptr(), f[i % R:].data_ptr(), sh) == 0


def grad(i):
    assert lib.exa_eval_grad(plans[i % R].handle, None, xs[i % R].data_ptr(), g[i % R].data_ptr(), sh) == 0


def graph_us(fn, n=64, reps=5):
    with torch.cuda.stream(st):
        for i in range(R):
            fn(i)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for i in range(n):
            fn(i)
    with torch.cuda.stream(st):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(reps):
            gr.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n)


if os.environ.get("EXA_NCU") == "1":
    with torch.cuda.stream(st):
        for i in range(2 * R):
            obj(i)
            grad(i)
    torch.cuda.synchronize()
    sys.exit(0)
lay = plans[0].layout
print(json.dumps({"workload": name, "obj_us": graph_us(obj), "grad_us": graph_us(grad),
                  "n_leaves": int(len(lay.leaves)), "n_prog": int(len(lay.prog)),
                  "n_obj_records": int(sum(tp.nrec for tp in model.plan.obj_terms))}), flush=True)
