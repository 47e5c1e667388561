#!/bin/bash
TAG=${1:-q27}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { m=$1; shift; env "$@" timeout 300 python tools/set_timing.py case13659 $m >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run set EXA_PDL=0
run set EXA_PDL=0 EXA_PREFETCH_TAB=0
run set EXA_PDL=1
run set EXA_PDL=1 EXA_THREADS=32
run set EXA_PDL=1 EXA_THREADS=32 EXA_PREFETCH_TAB=0
run set EXA_SEG_FILTER=heavy EXA_PDL=0
run set EXA_SEG_FILTER=heavy EXA_PDL=0 EXA_PREFETCH_TAB=0
EXA_TRACE=1 EXA_PDL=0 timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace.npz > gpurun_out/${TAG}.log 2>&1
echo done
