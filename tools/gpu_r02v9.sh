#!/bin/bash
# compressed set: re-sweep of the segmented sum's gathers per thread (grid size of the post-pass)
T=${1:-r02v9}
mkdir -p gpurun_out
for wl in case13659 case1354 mp96_case1354; do
  for ipt in 2 4 8 16; do
    echo -n "$wl ipt=$ipt "; EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py $wl 2>/dev/null | tail -1
  done
done | tee gpurun_out/${T}_cmp_ipt.txt
