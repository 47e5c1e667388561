#!/bin/bash
TAG=${1:-q30}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { w=$1; shift; env "$@" timeout 300 python tools/set_timing.py $w set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run case13659
run case13659 EXA_SC_TABLE=const
run case13659 EXA_SEG_FILTER=heavy
run case13659 EXA_SEG_FILTER=heavy EXA_SC_TABLE=const
run mp96_case1354 EXA_SC_TABLE=const
run mp96_case1354
EXA_TRACE=1 EXA_SC_TABLE=const timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace.npz > gpurun_out/${TAG}.log 2>&1
echo done
