"""Compressed callback set (exa_eval_set_compressed) timing at one workload:
set alone vs set + segmented sum, graph of rotating replicas.

    python tools/compressed_timing.py case13659 [R]
Prints one JSON line.  Under ncu (EXA_NCU=1) runs a few eager launches only.
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_12897_b200 import _lib, model_patterns
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import algorithmic_bytes, build_workload, eval_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
model = build_workload(name, lower_to_gpu=False)
a = algorithmic_bytes(model)
R = int(sys.argv[2]) if len(sys.argv) > 2 else max(3, int(np.ceil(2 * 126 * 2**20 / a["total"])))
dev = torch.device("cuda", 0)
plans = [DevicePlan(model, 0) for _ in range(R)]
jp, hp = model_patterns(model)
hj = [jp.device_handle(p, "jac") for p in plans]
hh = [hp.device_handle(p, "hess") for p in plans]
lib = _lib.load()
bufs = []
for r in range(R):
    x, y, w = eval_inputs(model, r)
    bufs.append(dict(x=torch.from_numpy(x).to(dev), y=torch.from_numpy(y).to(dev), w=w,
                     c=torch.empty(model.ncon, dtype=torch.float64, device=dev),
                     J=torch.empty(model.plan.n_jac_slots, dtype=torch.float64, device=dev),
                     H=torch.empty(model.plan.n_hess_slots, dtype=torch.float64, device=dev),
                     Jc=torch.empty(jp.nnz, dtype=torch.float64, device=dev),
                     Hc=torch.empty(hp.nnz, dtype=torch.float64, device=dev)))
st = torch.cuda.Stream(dev)
sh = C.c_void_p(st.cuda_stream)


def set_only(i):
    b, p = bufs[i % R], plans[i % R]
    assert lib.exa_eval_set(p.handle, None, b["x"].data_ptr(), b["y"].data_ptr(), b["w"], b["c"].data_ptr(),
                            b["J"].data_ptr(), b["H"].data_ptr(), sh) == 0


def comp(i, jpat=True, hpat=True):
    b, p = bufs[i % R], plans[i % R]
    assert lib.exa_eval_set_compressed(p.handle, None, hj[i % R] if jpat else None, hh[i % R] if hpat else None,
                                       b["x"].data_ptr(), b["y"].data_ptr(), b["w"], b["c"].data_ptr(),
                                       b["Jc"].data_ptr() if jpat else b["J"].data_ptr(),
                                       b["Hc"].data_ptr() if hpat else b["H"].data_ptr(), sh) == 0, \
        lib.exa_last_error()


WS = C.c_void_p()
assert lib.exa_workspace_create(plans[0].handle, C.byref(WS)) == 0


def comp_ws(i):
    """one workspace (one raw-slot scratch) for every replica, as a solver
    evaluating one model uses: inputs, parameters and outputs still rotate"""
    b, p = bufs[i % R], plans[i % R]
    assert lib.exa_eval_set_compressed(p.handle, WS, hj[i % R], hh[i % R], b["x"].data_ptr(), b["y"].data_ptr(),
                                       b["w"], b["c"].data_ptr(), b["Jc"].data_ptr(), b["Hc"].data_ptr(), sh) == 0


def graph_us(fn, n=8 * R, reps=5):
    with torch.cuda.stream(st):
        for i in range(R):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(n):
            fn(i)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n)


def graph_us_streams(n_streams, n=8 * R, reps=5):
    """comp() of replica r on stream r % n_streams (independent sets side by
    side; each plan's default workspace serves one stream)"""
    global sh
    sts = [st] + [torch.cuda.Stream(dev) for _ in range(n_streams - 1)]
    hs = [C.c_void_p(s.cuda_stream) for s in sts]

    def fn(i):
        global sh
        sh = hs[(i % R) % n_streams]
        comp(i)

    for i in range(R):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fork = torch.cuda.Event()
        fork.record(st)
        for s in sts[1:]:
            s.wait_event(fork)
        for i in range(n):
            fn(i)
        for s in sts[1:]:
            j = torch.cuda.Event()
            j.record(s)
            st.wait_event(j)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    sh = C.c_void_p(st.cuda_stream)
    return e0.elapsed_time(e1) * 1e3 / (reps * n)


if os.environ.get("EXA_NCU") == "1":
    with torch.cuda.stream(st):
        for i in range(2 * R):
            comp(i)
    torch.cuda.synchronize()
    sys.exit(0)
out = {"workload": name, "R": R, "set_us": graph_us(set_only), "set_comp_us": graph_us(comp),
       "set_comp_shared_ws_us": graph_us(comp_ws),
       "set_compJ_us": graph_us(lambda i: comp(i, True, False)),
       "set_compH_us": graph_us(lambda i: comp(i, False, True)),
       "set_comp_2streams_us": graph_us_streams(2), "set_comp_3streams_us": graph_us_streams(3),
       "nnz_jac": jp.nnz, "nnz_hess": hp.nnz, "env": {k: v for k, v in os.environ.items() if k.startswith("EXA_")}}
print(json.dumps(out), flush=True)
