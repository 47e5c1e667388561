#!/bin/bash
T=${1:-r02i}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -k "obj or compress" -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
for ipt in 8 4 8 4; do
  EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
done
EXA_CMP_IPT=8 timeout 600 python tools/compressed_timing.py mp96_case1354 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
EXA_CMP_IPT=4 timeout 600 python tools/compressed_timing.py mp96_case1354 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
timeout 600 python tools/obj_timing.py case13659 >> gpurun_out/${T}_obj.jsonl 2>> gpurun_out/${T}_obj.err
timeout 600 python tools/obj_timing.py mp96_case1354 >> gpurun_out/${T}_obj.jsonl 2>> gpurun_out/${T}_obj.err
EXA_NCU=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:compress -s 3 -c 1 -o gpurun_out/${T}_comp -f python tools/compressed_timing.py case13659 > gpurun_out/${T}_comp_ncu.log 2>&1
tail -2 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_comp.jsonl gpurun_out/${T}_obj.jsonl
