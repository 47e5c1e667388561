#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_GROUP_MAX=2
run EXA_GROUP_MAX=2 EXA_SPLIT=1
run EXA_GROUP_MAX=2 EXA_SPLIT=1 EXA_THREADS_HEAVY=64
run EXA_GROUP_MAX=4 EXA_SPLIT=1
run EXA_GROUP_MAX=1 EXA_SPLIT=1
run EXA_GROUP_MAX=2 EXA_SPLIT=1 EXA_RPT_LIGHT=2
echo done
