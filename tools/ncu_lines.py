"""Top CUDA source lines by warp-stall samples, with the dominant stall reasons.

    python tools/ncu_lines.py REPORT.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iw = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows[hi + 1:]:
    if r and r[0].isdigit():
        def f(i):
            try:
                return float(r[i])
            except ValueError:
                return 0.0
        lines.append((int(r[0]), r[1], f(iw), {nm: f(i) for i, nm in reasons}))
tot = sum(x[2] for x in lines) or 1
agg = {}
for _, _, _, rs in lines:
    for k, v in rs.items():
        agg[k] = agg.get(k, 0) + v
print("total samples", tot, "| by reason:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for ln, src, v, rs in sorted(lines, key=lambda x: -x[2])[:N]:
    top = ", ".join(f"{k} {x / v * 100:.0f}%" for k, x in sorted(rs.items(), key=lambda kv: -kv[1])[:3] if x)
    print(f"{v / tot * 100:5.1f}% L{ln}: {src.strip()[:90]:90s} [{top}]")
