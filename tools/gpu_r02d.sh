#!/bin/bash
T=${1:-r02d}
mkdir -p gpurun_out
timeout 600 python tools/compressed_timing.py case13659 > gpurun_out/${T}_comp.jsonl 2> gpurun_out/${T}_comp.err
EXA_PDL=0 timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
EXA_NCU=1 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_op_read.sum \
  -s 22 -c 8 --csv --log-file gpurun_out/${T}_comp_ncu.csv python tools/compressed_timing.py case13659 > gpurun_out/${T}_comp_ncu.log 2>&1
cat gpurun_out/${T}_comp.jsonl
