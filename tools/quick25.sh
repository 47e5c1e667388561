#!/bin/bash
TAG=${1:-q25}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { w=$1; m=$2; shift; shift; env "$@" timeout 300 python tools/set_timing.py $w $m >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
for w in case2000 case1354 case13659; do
run $w set EXA_SEG_FILTER=heavy EXA_PDL=0
run $w cons EXA_SEG_FILTER=heavy EXA_PDL=0
run $w set EXA_PDL=0
run $w set EXA_PDL=1
done
run case13659 set EXA_PDL=1 EXA_THREADS=32
run case13659 set EXA_PDL=0 EXA_THREADS=32
echo done
