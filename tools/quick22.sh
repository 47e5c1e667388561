#!/bin/bash
TAG=${1:-q22}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_SEG_FILTER=heavy EXA_ATTACH=0
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_GROUP_RPT=2
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_GROUP_RPT=2 EXA_MINB=8
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_GROUP_RPT=2 EXA_MINB=10
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_MINB=8
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_MINB=4
echo done
