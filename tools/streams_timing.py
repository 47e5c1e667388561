"""Independent callback sets on S concurrent streams (one fused launch per
set, each stream a PDL chain): us per set for S = 1, 2, 3, 4.

    python tools/streams_timing.py case13659
Prints one JSON line.  S = 1 is the bench's headline configuration; S > 1
runs S independent evaluation streams (several solver instances) side by side.
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_12897_b200 import _lib
from paper_2510_12897_b200.device import DevicePlan
from paper_2510_12897_b200.workloads import build_workload, eval_inputs, model_summary

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
model = build_workload(name, lower_to_gpu=False)
bps = model_summary(model)["bytes_per_set"]
R = max(4, int(np.ceil(2 * 126 * 2**20 / bps)))
R = (R + 11) // 12 * 12  # divisible by every S below
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
streams = [torch.cuda.Stream(dev) for _ in range(4)]


def launch(i, st):
    b = bufs[i % R]
    rc = lib.exa_eval_set(plans[i % R].handle, None, b[0].data_ptr(), b[1].data_ptr(), 1.0, b[2].data_ptr(),
                          b[3].data_ptr(), b[4].data_ptr(), C.c_void_p(st.cuda_stream))
    assert rc == 0, lib.exa_last_error()


def us_per_set(S, n=32 * 12, reps=5):
    main = streams[0]
    for i in range(R):
        launch(i, main)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        ev = torch.cuda.Event()
        ev.record(main)
        for s in streams[1:S]:
            s.wait_event(ev)
        for i in range(n):  # set i on stream i % S (replica i % R: S divides R)
            launch(i, streams[i % S])
        for s in streams[1:S]:
            e = torch.cuda.Event()
            e.record(s)
            main.wait_event(e)
    with torch.cuda.stream(main):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(main):
        e0.record(main)
        for _ in range(reps):
            g.replay()
        e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n)


out = {"workload": name, "bytes_per_set": bps, "R": R}
for S in (1, 2, 3, 4):
    us = us_per_set(S)
    out[f"S{S}"] = {"us_per_set": us, "sets_per_s": 1e6 / us, "GBps": bps / us / 1e3}
print(json.dumps(out), flush=True)
