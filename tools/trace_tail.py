"""Which tasks end last, per SM (trace_set.py output)."""
import sys
import numpy as np

d = np.load(sys.argv[1]); t = d["trace"]; segs = d["segs"]
sm, vb, c0, c1, g0, g1 = (t[:, i] for i in range(6))
G0 = g0.min(); gs = (g0 - G0) / 1e3; ge = (g1 - G0) / 1e3
sid = np.searchsorted(segs[:, 2], vb, side="right") - 1
ends = np.array([ge[sm == s].max() for s in range(sm.max() + 1)])
order = np.argsort(ends)[::-1]
print("slowest SMs: end | last task (seg, start, dur) | tasks on SM by seg")
for s in order[:10]:
    m = sm == s
    j = np.flatnonzero(m)[np.argmax(ge[m])]
    cnt = np.bincount(sid[m], minlength=len(segs))
    print(f"SM {s:3d} {ends[s]:.2f} | seg {sid[j]:2d} start {gs[j]:.2f} dur {ge[j]-gs[j]:.2f} | {cnt.tolist()}")
print("fastest SM:", order[-1], f"{ends[order[-1]]:.2f}", np.bincount(sid[sm == order[-1]], minlength=len(segs)).tolist())
# per segment: duration stats
for k in range(len(segs)):
    m = sid == k
    if m.any():
        dur = ge[m] - gs[m]
        print(f"seg {k:2d} n {m.sum():4d} dur mean {dur.mean():.2f} p90 {np.percentile(dur, 90):.2f} max {dur.max():.2f}")
