#!/bin/bash
T=${1:-r02g}
mkdir -p gpurun_out
for ipt in 4 8 12 16; do
  EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
done
for ipt in 8 16; do
  EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py mp96_case1354 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
done
for w in 0 64 256; do
  EXA_LOCALITY_W=$w timeout 900 python tools/set_timing.py n1_case2000 set >> gpurun_out/${T}_n1.jsonl 2>> gpurun_out/${T}_n1.err
done
EXA_THREADS=128 EXA_LOCALITY_W=64 timeout 900 python tools/set_timing.py n1_case2000 set >> gpurun_out/${T}_n1.jsonl 2>> gpurun_out/${T}_n1.err
EXA_THREADS=128 EXA_LOCALITY_W=0 timeout 900 python tools/set_timing.py n1_case2000 set >> gpurun_out/${T}_n1.jsonl 2>> gpurun_out/${T}_n1.err
cat gpurun_out/${T}_comp.jsonl gpurun_out/${T}_n1.jsonl
