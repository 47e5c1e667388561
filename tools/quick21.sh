#!/bin/bash
TAG=${1:-q21}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_SEG_FILTER=heavy
run EXA_SEG_FILTER=heavy EXA_MINB=12
run EXA_SEG_FILTER=heavy EXA_MINB=8
run EXA_SEG_FILTER=heavy EXA_ATTACH=0
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_GROUP_MAX=1
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_GROUP_MAX=4
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_SINCOS_IMPL=cuda
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_THREADS=32
run EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_THREADS=128
echo done
