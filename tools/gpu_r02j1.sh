#!/bin/bash
# direct compressed-Jacobian entries (compressed-set module): parity + timing
T=${1:-r02j1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -k "compress" -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for rep in 1 2; do
  for jd in 1 0; do
    for wl in case13659 mp96_case1354; do
      EXA_JDIRECT=$jd timeout 600 python tools/compressed_timing.py $wl >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
    done
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02j1_comp.jsonl"):
    d = json.loads(l); print(d["workload"], d["env"].get("EXA_JDIRECT"), "set", round(d["set_us"], 2), "comp", round(d["set_comp_us"], 2), "shared_ws", round(d["set_comp_shared_ws_us"], 2), "J", round(d["set_compJ_us"], 2), "H", round(d["set_compH_us"], 2))
PY
