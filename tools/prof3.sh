#!/bin/bash
TAG=${1:-p}
EXA_R=1 EXA_SEG_FILTER=heavy timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:exa_k_set -s 12 -c 1 \
  -o gpurun_out/${TAG}_heavy -f python tools/set_timing.py case13659 set > gpurun_out/${TAG}_prof.log 2>&1
echo done
