#!/bin/bash
TAG=${1:-q24}
mkdir -p gpurun_out
./tools/micro/sincos_bench > gpurun_out/${TAG}_sincos.txt 2>&1
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { m=$1; shift; env "$@" timeout 300 python tools/set_timing.py case13659 $m >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run set EXA_PDL=0
run set EXA_PDL=1
run set EXA_SEG_FILTER=heavy EXA_PDL=0
run set EXA_PDL=1 EXA_BUCKETS=0 EXA_ATTACH=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo done
