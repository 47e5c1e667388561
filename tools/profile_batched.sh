#!/bin/bash
# ncu captures of the set kernel on the batched configs (run under gpurun)
TAG=${1:-p}
mkdir -p gpurun_out
for w in mp96_case1354 n1_case2000; do
  timeout 900 ncu --set full --clock-control none -k regex:exa_k_set -s 3 -c 1 \
    -o gpurun_out/${TAG}_prof_${w} -f python tools/set_timing.py $w set > gpurun_out/${TAG}_ncu_${w}.log 2>&1
done
echo done
