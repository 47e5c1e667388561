#!/bin/bash
# Steady-state DRAM bytes per set of ONE workload (see tools/ncu_steady.sh):
#   bash tools/ncu_steady_one.sh TAG WORKLOAD R
T=${1:-r02}; W=${2:-n1_case2000}; R=${3:-3}
mkdir -p gpurun_out
EXA_R=$R timeout 1500 ncu --graph-profiling graph --clock-control none --cache-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
  -s $(( R + 3 )) -c 2 --csv --log-file gpurun_out/${T}_steady_${W}.csv \
  python tools/set_timing.py $W set > gpurun_out/${T}_steady_${W}.log 2>&1
echo done
