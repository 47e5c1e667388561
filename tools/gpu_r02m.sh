#!/bin/bash
T=${1:-r02m}
mkdir -p gpurun_out
for gm in auto 1 2 4; do
  EXA_GROUP_MAX=$gm timeout 300 python tools/set_timing.py case1354 set >> gpurun_out/${T}_c1354.jsonl 2>> gpurun_out/${T}_c1354.err
done
for gm in 1 2; do
  EXA_GROUP_MAX=$gm EXA_SEG_ORDER=BOG timeout 300 python tools/set_timing.py case1354 set >> gpurun_out/${T}_c1354.jsonl 2>> gpurun_out/${T}_c1354.err
done
cat gpurun_out/${T}_c1354.jsonl
