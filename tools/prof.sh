#!/bin/bash
# ncu full capture of one set-kernel launch and one cons-kernel launch
TAG=${1:-p}
W=${2:-case13659}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exa_k_set -s 12 -c 1 \
  -o gpurun_out/${TAG}_set -f python tools/set_timing.py $W set > gpurun_out/${TAG}_prof.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:exa_k_cons -s 12 -c 1 \
  -o gpurun_out/${TAG}_cons -f python tools/set_timing.py $W cons >> gpurun_out/${TAG}_prof.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:exa_k_hess -s 12 -c 1 \
  -o gpurun_out/${TAG}_hess -f python tools/set_timing.py $W hess >> gpurun_out/${TAG}_prof.log 2>&1
echo done
