#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
for w in case14 case1354 case2000 case13659; do
  for f in heavy light all; do
    EXA_SEG_FILTER=$f timeout 300 python tools/set_timing.py $w set >> $OUT 2>> gpurun_out/${TAG}_timing.err
  done
done
echo done
