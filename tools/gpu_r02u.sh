#!/bin/bash
# A/B of the sin/cos table L1 prefetch (EXA_SC_PF), interleaved runs
T=${1:-r02u}
mkdir -p gpurun_out
for rep in 1 2; do
  for pf in 0 1; do
    for wl in case13659 mp96_case1354 case1354; do
      EXA_SC_PF=$pf timeout 300 python tools/set_timing.py $wl >> gpurun_out/${T}_sc.jsonl 2>> gpurun_out/${T}_sc.err
    done
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02u_sc.jsonl"):
    d = json.loads(l); print(d.get("workload"), d.get("env", {}).get("EXA_SC_PF"), round(d.get("us_per_set", d.get("us", 0)), 3))
PY
