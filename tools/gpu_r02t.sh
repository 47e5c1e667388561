#!/bin/bash
# compressed set with raw J / H kept in L2 (exa_k_setk_*), vs evict-first raw stores
T=${1:-r02t}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -k "compress" -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
for k in 1 0; do
  for wl in case13659 mp96_case1354 case1354; do
    EXA_SETK=$k timeout 600 python tools/compressed_timing.py $wl >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
  done
done
tail -2 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_comp.jsonl
