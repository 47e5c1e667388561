#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
timeout 300 python tools/split_timing.py >> $OUT 2>> gpurun_out/${TAG}_timing.err
for mb in 5 6 7 8; do EXA_MINB=$mb timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; done
EXA_PDL=0 EXA_SPLIT=1 timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err
echo done
