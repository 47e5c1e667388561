#!/bin/bash
TAG=${1:-q18}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_PERSIST=0
run EXA_PERSIST=0 EXA_BUCKETS=0
EXA_TRACE=1 EXA_PERSIST=0 timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace_classic.npz > gpurun_out/${TAG}.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo done
