#!/bin/bash
TAG=${1:-q34}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { w=$1; shift; env "$@" timeout 300 python tools/set_timing.py $w set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run case13659
run case13659 EXA_SEG_FILTER=heavy
run mp96_case1354
run n1_case2000
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
EXA_TRACE=1 timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace.npz > gpurun_out/${TAG}.log 2>&1
echo done
