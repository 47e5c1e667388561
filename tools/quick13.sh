#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_THREADS=64
run EXA_THREADS=32
run EXA_SPLIT=1 EXA_THREADS_HEAVY=32
run EXA_SPLIT=1 EXA_THREADS_HEAVY=64
run EXA_SPLIT=1 EXA_THREADS_HEAVY=32 EXA_GROUP_MAX=1
run EXA_SEG_FILTER=heavy EXA_THREADS=32
run EXA_SEG_FILTER=heavy EXA_THREADS=64
run EXA_SEG_FILTER=heavy EXA_THREADS=32 EXA_GROUP_MAX=1
run EXA_SEG_FILTER=heavy EXA_THREADS=32 EXA_GROUP_MAX=4
echo done
