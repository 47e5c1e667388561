#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_R=1
run EXA_R=2
run EXA_R=4
run EXA_R=11
run EXA_R=1 EXA_SEG_FILTER=heavy
run EXA_R=11 EXA_SEG_FILTER=heavy
run EXA_R=1 EXA_SEG_FILTER=light
echo done
