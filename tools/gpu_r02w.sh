#!/bin/bash
# many-wave set kernel knobs at N-1 and MP96 (us per set, graph of rotating replicas)
T=${1:-r02w}
mkdir -p gpurun_out
run() {  # env... -- workload
  env "$@" timeout 600 python tools/set_timing.py ${WL} >> gpurun_out/${T}_sweep.jsonl 2>> gpurun_out/${T}_sweep.err
}
for WL in n1_case2000 mp96_case1354; do
  run EXA_X=base
  run EXA_GROUP_RPT=2
  run EXA_GROUP_MAX=4
  run EXA_GROUP_MAX=1
  run EXA_THREADS=128
  run EXA_MINB=3
  run EXA_ST_CS=0
done
python - <<'PY'
import json
for l in open("gpurun_out/r02w_sweep.jsonl"):
    d = json.loads(l); print(d.get("workload"), {k: v for k, v in d.get("env", {}).items()}, round(d.get("us_per_set", 0), 2), d.get("regs"))
PY
