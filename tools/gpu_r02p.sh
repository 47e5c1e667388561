#!/bin/bash
T=${1:-r02p}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -k "compress" -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
for ipt in 4 8 2; do
  EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
done
EXA_CMP_IPT=4 timeout 600 python tools/compressed_timing.py mp96_case1354 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
tail -2 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_comp.jsonl
