"""Summarise a trace_set.py timeline: per-segment durations, SM busy time."""
import sys
import numpy as np

d = np.load(sys.argv[1])
t = d["trace"]
segs = d["segs"]
sm, vb, c0, c1, g0, g1 = (t[:, i] for i in range(6))
ok = c1 > 0
print("records", ok.sum(), "of", len(t))
G0 = g0[ok].min()
gs, ge = (g0 - G0) / 1e3, (g1 - G0) / 1e3
print(f"globaltimer span: {ge[ok].max():.2f} us;  start spread {gs[ok].min():.2f}..{gs[ok].max():.2f}")
dur = (c1 - c0) / 1965.0  # us at 1965 MHz
# segment of each vb
starts = segs[:, 2]
sid = np.searchsorted(starts, vb, side="right") - 1
kinds = {0: "term", 1: "row", 2: "fold", 3: "group", 4: "bkt", 5: "pair"}
print("seg  term kind   nvb   warp-dur mean/max us   start min/max us   end max us")
for s in range(len(segs)):
    m = ok & (sid == s)
    if not m.any():
        continue
    print(f"{s:3d} {segs[s,0]:4d} {kinds[segs[s,1] & 15]:3s}{segs[s,1] >> 4:2d} {len(np.unique(vb[m])):5d}   {dur[m].mean():6.2f} {dur[m].max():6.2f}"
          f"   {gs[m].min():7.2f} {gs[m].max():7.2f}   {ge[m].max():7.2f}")
# per-SM: first start, last end (globaltimer)
print("per-SM last end (us): min %.2f median %.2f max %.2f" % tuple(
    np.percentile([ge[ok & (sm == k)].max() for k in np.unique(sm[ok])], [0, 50, 100])))
print("per-SM first start (us): min %.2f median %.2f max %.2f" % tuple(
    np.percentile([gs[ok & (sm == k)].min() for k in np.unique(sm[ok])], [0, 50, 100])))
# concurrency histogram over time (warps in flight)
# phase stamps (lane 0, clock64 relative to the warp start), where recorded
ph = t[:, 6:10]
for s in range(len(segs)):
    m = ok & (sid == s) & (ph[:, 0] > 0)
    if not m.any():
        continue
    rel = [(ph[m, k] - c0[m]) / 1965.0 for k in range(3)]
    print(f"seg {s:3d} phases (us from warp start): loads {rel[0].mean():.2f}  gathers {rel[1].mean():.2f}"
          f"  p2 {rel[2][ph[m, 2] > 0].mean() if (ph[m, 2] > 0).any() else float('nan'):.2f}  end {dur[m].mean():.2f}")
T = np.linspace(0, ge[ok].max(), 40)
conc = [((gs[ok] <= x) & (ge[ok] > x)).sum() for x in T]
print("warps in flight over time:", " ".join(str(c) for c in conc))
