#!/bin/bash
TAG=${1:-q29}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { w=$1; shift; env "$@" timeout 300 python tools/set_timing.py $w set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
for w in n1_case2000 mp96_case1354; do
for t in 32 64 128 256; do run $w EXA_THREADS=$t; done
run $w EXA_THREADS=128 EXA_PDL=0
done
echo done
