#!/bin/bash
# single-instance sets: CTA size (threads) re-check, interleaved
T=${1:-r02c2}
mkdir -p gpurun_out
for rep in 1 2; do
  for wl in case13659 case1354; do
    for th in auto 64 128; do
      EXA_THREADS=$th timeout 600 python tools/set_timing.py $wl >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
    done
  done
done
EXA_SHARD=0/4 timeout 600 python tools/set_timing.py mp96_case1354 >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
EXA_SHARD=0/4 EXA_THREADS=128 timeout 600 python tools/set_timing.py mp96_case1354 >> gpurun_out/${T}.jsonl 2>> gpurun_out/${T}.err
python - <<'PY'
import json
for l in open("gpurun_out/r02c2.jsonl"):
    d = json.loads(l); print(d.get("workload"), {k: v for k, v in d.get("env", {}).items()}, round(d.get("us_per_set", 0), 3), d.get("ctas", {}).get("set_l"), d.get("ctas", {}).get("set_h"))
PY
