#!/bin/bash
# ncu full capture of the set kernel with dense warp sampling (source-level stalls)
TAG=${1:-p5}
mkdir -p gpurun_out
EXA_R=3 timeout 900 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:exa_k_set -s 20 -c 1 \
  -o gpurun_out/${TAG}_set -f python tools/set_timing.py case13659 set > gpurun_out/${TAG}_prof.log 2>&1
echo done
