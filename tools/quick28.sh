#!/bin/bash
TAG=${1:-q28}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { m=$1; shift; env "$@" timeout 300 python tools/set_timing.py case13659 $m >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run set EXA_PDL=1
run set EXA_PDL=1 EXA_PDL_EARLY=1
run set EXA_PDL=1 EXA_PDL_EARLY=1 EXA_THREADS=64
run set EXA_PDL=1 EXA_PDL_EARLY=1 EXA_GROUP_MAX=4
run set EXA_PDL=1 EXA_GROUP_MAX=4
run set EXA_PDL=1 EXA_PDL_EARLY=1 EXA_MINB=16
echo done
