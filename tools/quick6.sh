#!/bin/bash
TAG=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
for gm in 4 2 1; do EXA_GROUP_MAX=$gm timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; done
EXA_GROUP_MAX=4 EXA_SEG_FILTER=heavy timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err
EXA_GROUP_MAX=4 EXA_THREADS=128 timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err
echo done
