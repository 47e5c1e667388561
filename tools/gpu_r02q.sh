#!/bin/bash
T=${1:-r02q}
mkdir -p gpurun_out
EXA_CMP_PROBE=1 timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
EXA_CMP_PROBE=1 EXA_CMP_IPT=16 timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
EXA_CMP_PROBE=1 timeout 600 python tools/compressed_timing.py mp96_case1354 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
cat gpurun_out/${T}_comp.jsonl
