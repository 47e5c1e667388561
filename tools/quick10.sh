#!/bin/bash
TAG=${1:-q}
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
for f in light fold aug other; do run EXA_SEG_FILTER=$f; done
for f in light fold aug other; do run EXA_SEG_FILTER=$f EXA_R=1; done
echo done
