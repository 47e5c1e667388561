#!/bin/bash
# persistent-kernel sweep: correctness first, then timings
TAG=${1:-q15}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_PERSIST=0
run EXA_PERSIST=4
run EXA_PERSIST=4 EXA_PDL=0
run EXA_PERSIST=4 EXA_MINB=4
run EXA_PERSIST=2
run EXA_PERSIST=2 EXA_MINB=8
run EXA_PERSIST=8
run EXA_PERSIST=8 EXA_MINB=2
run EXA_PERSIST=16
run EXA_PERSIST=4 EXA_THREADS=32
run EXA_PERSIST=2 EXA_THREADS=128
echo done
