#!/bin/bash
# quick GPU check: tests + timing of each callback mode
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
for m in set cons jac hess; do timeout 300 python tools/set_timing.py ${2:-case13659} $m >> $OUT 2>> gpurun_out/${TAG}_timing.err; done
echo done
