#!/bin/bash
# ncu full capture of the set kernel (case13659), steady-state launch
TAG=${1:-p4}
mkdir -p gpurun_out
EXA_R=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:exa_k_set -s 20 -c 1 \
  -o gpurun_out/${TAG}_set -f python tools/set_timing.py case13659 set > gpurun_out/${TAG}_prof.log 2>&1
echo done
