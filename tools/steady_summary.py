"""Steady-state DRAM bytes per set from tools/ncu_steady.sh's csv files
(ncu --graph-profiling graph over a CUDA graph of 64 x R rotating-replica
set launches; per-set bytes = graph bytes / (64 R)), written as
profiles/<TAG>_steady_ncu_summary_<workload>.json -- bench.py's
roofline.traffic reads them (run here, no GPU).

    python tools/steady_summary.py TAG
"""
import csv
import io
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
for workload, R in (("case13659", 11), ("mp96_case1354", 3), ("n1_case2000", 3)):
    src = ROOT / "profiles" / f"{TAG}_steady_ncu_{workload}.csv"
    if not src.is_file():
        continue
    lines = src.read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    per = {}
    for row in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        per.setdefault(row["ID"], {})[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
    n = 64 * R
    rd = statistics.mean(v["dram__bytes_read.sum"] for v in per.values()) / n
    wr = statistics.mean(v["dram__bytes_write.sum"] for v in per.values()) / n
    out = {"tag": TAG, "workload": workload, "sets_per_graph": n, "graph_replays_profiled": len(per),
           "steady_state_dram_bytes_per_set": rd + wr, "dram_read_bytes_per_set": rd, "dram_write_bytes_per_set": wr,
           "source": src.name,
           "note": "ncu --graph-profiling graph --cache-control none over CUDA-graph replays of back-to-back set "
                   "launches on rotating replicas (tools/ncu_steady.sh): the L2 state between sets is the "
                   "benchmark's, not a cold single launch's"}
    dst = ROOT / "profiles" / f"{TAG}_steady_ncu_summary_{workload}.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(dst.name, round((rd + wr) / 1e6, 2), "MB per set")
