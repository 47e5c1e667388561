#!/bin/bash
TAG=${1:-v2}
OUT=gpurun_out/${TAG}_variants.jsonl
: > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 >> $OUT 2>> gpurun_out/${TAG}_variants.err; }
run EXA_THREADS=256
run EXA_THREADS=128
run EXA_THREADS=512
run EXA_THREADS=256 EXA_MINB=5
run EXA_THREADS=256 EXA_SINCOS_IMPL=cuda
bash tools/prof.sh $TAG
echo done
