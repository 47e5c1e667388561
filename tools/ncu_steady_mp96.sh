T=r02h
cfg="mp96_case1354 3"
set -- $cfg
EXA_R=$2 timeout 1200 ncu --graph-profiling graph --clock-control none --cache-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
  -s $(( $2 + 3 )) -c 2 --csv --log-file gpurun_out/${T}_steady_$1.csv \
  python tools/set_timing.py $1 set > gpurun_out/${T}_steady_$1.log 2>&1
echo done
