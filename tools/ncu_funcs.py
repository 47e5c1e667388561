"""Per-function totals (instructions executed, warp-stall samples) of a
generated module from an ncu report captured with --import-source on.

    python tools/ncu_funcs.py REPORT.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]


def page(view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


full = page("cuda")
hi = next(i for i, r in enumerate(full) if r and r[0] == "Line No")
text = {int(r[0]): r[1] for r in full[hi + 1:] if r and r[0].isdigit()}
func_of, cur = {}, "prelude"
for ln in sorted(text):
    m = re.match(r'\s*(?:template <int MODE>\s*)?(?:extern "C" )?(?:EXA_FN|__device__|__global__)[^(]*?\b(\w+)\s*\(', text[ln])
    if m:
        cur = m.group(1)
    func_of[ln] = cur
rows = page("cuda,sass")
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ie, iw = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = {}
for r in rows[hi + 1:]:
    if r and r[0].isdigit():
        f = func_of.get(int(r[0]), "?")
        a = agg.setdefault(f, [0.0, 0.0])
        for j, i in enumerate((ie, iw)):
            try:
                a[j] += float(r[i])
            except ValueError:
                pass
ti = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti:.0f}, stall samples {tw:.0f}")
for f, (i, w) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{f:36s} instr {i:9.0f} ({i / ti * 100:4.1f}%)  stalls {w / tw * 100:4.1f}%")
