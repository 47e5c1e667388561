#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_THREADS=64 EXA_GROUP_MAX=4
run EXA_THREADS=64 EXA_GROUP_MAX=1
run EXA_THREADS=96
run EXA_THREADS=128
run EXA_THREADS=64 EXA_MINB=10
run EXA_THREADS=64 EXA_RPT_LIGHT=2
run EXA_THREADS=64
echo done
