#!/bin/bash
# keyed per-element parameter columns (N-1): GPU parity + timing A/B
T=${1:-r02p2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for rep in 1 2; do
  for pp in 1 0; do
    EXA_PERIODIC=$pp timeout 900 python tools/set_timing.py n1_case2000 >> gpurun_out/${T}_t.jsonl 2>> gpurun_out/${T}_t.err
  done
done
EXA_PERIODIC=1 timeout 600 python tools/set_timing.py mp96_case1354 >> gpurun_out/${T}_t.jsonl 2>> gpurun_out/${T}_t.err
python - <<'PY'
import json
for l in open("gpurun_out/r02p2_t.jsonl"):
    d = json.loads(l); print(d["workload"], d["env"], round(d["us_per_set"], 2), d.get("bytes"), round(d.get("GBps", 0)))
PY
