#!/bin/bash
TAG=${1:-q33}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { w=$1; shift; env "$@" timeout 300 python tools/set_timing.py $w set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run case13659
run case13659 EXA_GROUP_MAX=1
run case13659 EXA_ATTACH=0
run case13659 EXA_GROUP_MAX=1 EXA_SEG_FILTER=heavy
run case13659 EXA_SEG_FILTER=heavy
run case13659 EXA_THREADS=64
echo done
