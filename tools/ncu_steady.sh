#!/bin/bash
# Steady-state DRAM bytes per set: ncu profiles whole CUDA-graph replays
# (--graph-profiling graph) of S x R back-to-back set launches on rotating
# replicas (tools/set_timing.py), so L2 state between sets is the bench's,
# not a cold single launch's.  Per-set bytes = graph bytes / (S x R).
# Skips the R eager warm-up launches and 3 warm-up replays, profiles 2 replays.
T=${1:-r02}
mkdir -p gpurun_out
for cfg in "case13659 11" "mp96_case1354 3" "n1_case2000 3"; do
  set -- $cfg
  EXA_R=$2 timeout 1200 ncu --graph-profiling graph --clock-control none --cache-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    -s $(( $2 + 3 )) -c 2 --csv --log-file gpurun_out/${T}_steady_$1.csv \
    python tools/set_timing.py $1 set > gpurun_out/${T}_steady_$1.log 2>&1
done
echo done
