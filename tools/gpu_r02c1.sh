#!/bin/bash
# small shards (MP96 / N-1 split 8 ways): CTA size and grouping knobs
T=${1:-r02c1}
mkdir -p gpurun_out
for wl in mp96_case1354 n1_case2000; do
  for cfg in "auto auto" "32 auto" "32 4" "128 auto" "256 4" "64 auto"; do
    set -- $cfg
    EXA_SHARD=0/8 EXA_THREADS=$1 EXA_GROUP_MAX=$2 timeout 600 python tools/set_timing.py $wl >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02c1.jsonl"):
    d = json.loads(l); print(d.get("workload"), {k: v for k, v in d.get("env", {}).items()}, round(d.get("us_per_set", 0), 2), d.get("ctas", {}).get("set_l"), d.get("ctas", {}).get("set_h"))
PY
