"""Time the KKT assembly (exa_kkt_values) at case13659 on the GPU.

    python tools/kkt_timing.py [workload]
Prints one JSON line: entries, us per assembly, algorithmic GB/s
(8-B descriptor + gathered value(s) + 8-B store per entry).
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2510_12897_b200.kkt import KKTSystem
from paper_2510_12897_b200.workloads import build_workload

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
model = build_workload(name, lower_to_gpu=False)
ks = KKTSystem(model)
dev = torch.device("cuda", 0)
R = 8  # rotating replicas (> L2)
reps = []
for r in range(R):
    reps.append((torch.rand(ks.hpat.nnz, dtype=torch.float64, device=dev),
                 torch.rand(ks.jpat.nnz, dtype=torch.float64, device=dev),
                 torch.rand(ks.nz, dtype=torch.float64, device=dev),
                 torch.empty(ks.nnz, dtype=torch.float64, device=dev)))
for h, j, s, o in reps:
    ks.values(h, j, s, 1e-8, 0.0, out=o)
torch.cuda.synchronize()
# one CUDA graph of N assemblies (no Python overhead inside the timed region)
N = 8 * R
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for i in range(N):
            h, j, s, o = reps[i % R]
            ks.values(h, j, s, 1e-8, 0.0, out=o)
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(10):
        g.replay()
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (10 * N)
kind = (ks.desc[:, 0].astype(np.int64) & 0xFFFFFFFF) >> 29
reads = 8 * ks.nnz + 8 * int(np.isin(kind, (0, 1, 3)).sum()) + 8 * int(np.isin(kind, (1, 2)).sum())
bytes_ = reads + 8 * ks.nnz
print(json.dumps({"workload": name, "kkt_entries": ks.nnz, "n": ks.n, "us_per_assembly": us,
                  "algorithmic_bytes": bytes_, "GBps": bytes_ / us / 1e3}))
