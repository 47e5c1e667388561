#!/bin/bash
TAG=${1:-v4}
OUT=gpurun_out/${TAG}_variants.jsonl
: > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 >> $OUT 2>> gpurun_out/${TAG}_variants.err; }
run EXA_SEG_FILTER=heavy
run EXA_SEG_FILTER=light
run EXA_SEG_FILTER=heavy EXA_SINCOS_IMPL=cuda
run EXA_SEG_FILTER=light EXA_THREADS=128
echo done
