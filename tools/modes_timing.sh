#!/bin/bash
# per-callback kernels vs the fused set (run under gpurun)
TAG=${1:-m}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_modes.jsonl; : > $OUT
for w in case13659 mp96_case1354; do
  for m in set cons jac hess; do timeout 300 python tools/set_timing.py $w $m >> $OUT 2>> gpurun_out/${TAG}_modes.err; done
done
echo done
