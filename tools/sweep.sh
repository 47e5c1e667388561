#!/bin/bash
# Timing sweep of set-kernel variants (env knobs of jit.py / device.py), one
# JSON line each:   tools/sweep.sh TAG WORKLOAD "ENV1=a ENV2=b" "ENV1=c" ...
TAG=$1; W=$2; shift 2
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
for v in "" "$@"; do
  env $v timeout 300 python tools/set_timing.py $W set >> $OUT 2>> gpurun_out/${TAG}_timing.err
done
echo done
