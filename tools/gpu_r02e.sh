#!/bin/bash
T=${1:-r02e}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -k "compress" -q -p no:cacheprovider > gpurun_out/${T}_cmp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_cmp_tests.log
timeout 600 python tools/compressed_timing.py case13659 > gpurun_out/${T}_comp.jsonl 2> gpurun_out/${T}_comp.err
EXA_ST_CS=0 timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
timeout 600 python tools/compressed_timing.py mp96_case1354 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
EXA_NCU=1 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_read.sum \
  -k regex:compress -s 11 -c 4 --csv --log-file gpurun_out/${T}_comp_ncu.csv python tools/compressed_timing.py case13659 > gpurun_out/${T}_comp_ncu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -2 gpurun_out/${T}_cmp_tests.log
cat gpurun_out/${T}_comp.jsonl
