#!/bin/bash
TAG=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_GROUP_MAX=2
run EXA_GROUP_MAX=2 EXA_SPLIT=1
run EXA_GROUP_MAX=4 EXA_SPLIT=1
run EXA_GROUP_MAX=1 EXA_SPLIT=1
run EXA_GROUP_MAX=2 EXA_SEG_FILTER=heavy
run EXA_R=1 EXA_GROUP_MAX=2 EXA_SEG_FILTER=heavy
echo done
