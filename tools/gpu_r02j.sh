#!/bin/bash
T=${1:-r02j}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_edge.py -k "obj or compress" -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
for ipt in 8 4 16; do
  EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
done
timeout 600 python tools/obj_timing.py case13659 >> gpurun_out/${T}_obj.jsonl 2>> gpurun_out/${T}_obj.err
timeout 600 python tools/obj_timing.py mp96_case1354 >> gpurun_out/${T}_obj.jsonl 2>> gpurun_out/${T}_obj.err
for v in 0 1 0 1; do
  EXA_PRE_WAIT_CONST=$v timeout 300 python tools/set_timing.py case13659 set >> gpurun_out/${T}_prewait.jsonl 2>> gpurun_out/${T}_prewait.err
done
EXA_PRE_WAIT_CONST=1 timeout 300 python tools/set_timing.py mp96_case1354 set >> gpurun_out/${T}_prewait.jsonl 2>> gpurun_out/${T}_prewait.err
tail -2 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_comp.jsonl gpurun_out/${T}_obj.jsonl gpurun_out/${T}_prewait.jsonl
