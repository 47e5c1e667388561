#!/bin/bash
# timing sweep of kernel-configuration knobs; output gpurun_out/$1_variants.jsonl
TAG=${1:-exp}
OUT=gpurun_out/${TAG}_variants.jsonl
: > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 >> $OUT 2>> gpurun_out/${TAG}_variants.err; }
run EXA_THREADS=256
run EXA_THREADS=128
run EXA_THREADS=256 EXA_MINB=5
run EXA_THREADS=256 EXA_MINB=6
run EXA_THREADS=128 EXA_MINB=12
run EXA_THREADS=256 EXA_SINCOS_IMPL=cuda
run EXA_THREADS=128 EXA_SINCOS_IMPL=cuda
for m in cons jac hess; do env EXA_THREADS=256 timeout 300 python tools/set_timing.py case13659 $m >> $OUT 2>> gpurun_out/${TAG}_variants.err; done
echo done
