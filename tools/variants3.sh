#!/bin/bash
TAG=${1:-v3}
OUT=gpurun_out/${TAG}_variants.jsonl
: > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 >> $OUT 2>> gpurun_out/${TAG}_variants.err; }
run EXA_RPT_LIGHT=1
run EXA_RPT_LIGHT=2
run EXA_RPT_LIGHT=4
run EXA_RPT_LIGHT=8
run EXA_RPT_LIGHT=4 EXA_THREADS=128
echo done
