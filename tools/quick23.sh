#!/bin/bash
TAG=${1:-q23}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { m=$1; shift; env "$@" timeout 300 python tools/set_timing.py case13659 $m >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
for m in set cons jac hess; do
run $m EXA_SEG_FILTER=heavy EXA_ATTACH=0
run $m EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_SINCOS_IMPL=cuda
done
run set EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_THREADS=32 EXA_MINB=32
run set EXA_SEG_FILTER=heavy EXA_ATTACH=0 EXA_THREADS=32 EXA_MINB=24
echo done
