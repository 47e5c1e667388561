"""Summarise an ncu launch list + full capture into profiles/ (run here, no GPU).

    python tools/summarize_ncu.py TAG WORKLOAD  [gpurun_out/TAG_launches.csv gpurun_out/TAG_prof_set.ncu-rep]

Writes profiles/<TAG>_ncu_summary.json (read by bench.py for roofline.traffic)
and profiles/<TAG>_launches.csv (the per-launch duration list, trimmed).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_write.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "nsecond": 1e-9, "msecond": 1e-3}


def raw_metrics(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            if h in WANT or h == "Kernel Name":
                try:
                    d[h] = float(v.replace(",", "")) * UNIT.get(u, 1.0) if h != "Kernel Name" else v
                except ValueError:
                    d[h] = v
        stalls = {}
        for h, v in zip(hdr, vals):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        launches.append(d)
    return launches


def launch_list(path: Path):
    lines = [ln for ln in path.read_text().splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            scale = UNIT.get(r["Metric Unit"], 1.0)
            per[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")) * scale)
    total = sum(sum(v) for v in per.values())
    return rows, {k: {"launches": len(v), "mean_us": 1e6 * sum(v) / len(v), "share": sum(v) / total}
                  for k, v in per.items()}


def main():
    tag, workload = sys.argv[1], sys.argv[2]
    lcsv = Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / f"gpurun_out/{tag}_launches.csv"
    rep = Path(sys.argv[4]) if len(sys.argv) > 4 else ROOT / f"gpurun_out/{tag}_prof_set.ncu-rep"
    rows, shares = launch_list(lcsv)
    full = raw_metrics(rep)
    from paper_2510_12897_b200.workloads import build_workload, model_summary

    bps = model_summary(build_workload(workload, lower_to_gpu=False))["bytes_per_set"]
    k = full[0]
    dram = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    summary = {
        "tag": tag, "workload": workload, "kernel": k.get("Kernel Name"),
        "algorithmic_bytes_per_launch": bps,
        "dram_bytes_per_launch": dram,
        "dram_read_bytes": k.get("dram__bytes_read.sum"), "dram_write_bytes": k.get("dram__bytes_write.sum"),
        "note": ("ncu replays with flushed caches and serialised launches: the absolute duration is "
                 "cold-cache; the kernel's share of the launch list is what compares with bench.py. "
                 "Writes are absorbed by the 126 MB L2 within one launch (write-back), so DRAM write "
                 "bytes per launch under-count the steady-state write traffic."),
        "full_capture": full,
        "launch_list_shares": shares,
    }
    out = ROOT / "profiles" / f"{tag}_ncu_summary.json"
    out.write_text(json.dumps(summary, indent=1))
    (ROOT / "profiles" / f"{tag}_launches.csv").write_text(
        "kernel,grid,block,duration_ns\n" + "\n".join(
            f'{r["Kernel Name"]},{r["Grid Size"].replace(",", " ")},{r["Block Size"].replace(",", " ")},{r["Metric Value"]}'
            for r in rows if r.get("Metric Name") == "gpu__time_duration.sum") + "\n")
    print(json.dumps({k2: v for k2, v in summary.items() if k2 != "full_capture"}, indent=1))


if __name__ == "__main__":
    main()
