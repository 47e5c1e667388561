#!/bin/bash
# periodic parameter columns (MP / scenario models): GPU parity + timing A/B
T=${1:-r02p1}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for rep in 1 2; do
  for pp in 1 0; do
    for wl in mp96_case1354 scen96_case1354; do
      EXA_PERIODIC=$pp timeout 600 python tools/set_timing.py $wl >> gpurun_out/${T}_t.jsonl 2>> gpurun_out/${T}_t.err
    done
    EXA_PERIODIC=$pp EXA_SHARD=0/8 timeout 600 python tools/set_timing.py mp96_case1354 >> gpurun_out/${T}_t.jsonl 2>> gpurun_out/${T}_t.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02p1_t.jsonl"):
    d = json.loads(l); print(d["workload"], d["env"], round(d["us_per_set"], 2), d.get("bytes"), d.get("GBps"))
PY
