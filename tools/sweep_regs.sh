#!/bin/bash
# register cap / sin-cos slow-path placement sweep of the fused set kernel
T=${1:-r02s}
OUT=gpurun_out/${T}_regs.jsonl; : > $OUT
for cfg in "32 0" "32 1" "24 1" "20 0" "20 1" "16 0" "16 1"; do
  set -- $cfg
  EXA_MINB=$1 EXA_SC_SLOW_INLINE=$2 timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${T}_regs.err
done
for cfg in "32 1" "20 1" "16 1"; do
  set -- $cfg
  EXA_EXACT_ZERO_SIGN=1 EXA_MINB=$1 EXA_SC_SLOW_INLINE=$2 timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${T}_regs.err
done
for cfg in "4 0" "4 1" "3 1" "2 1"; do
  set -- $cfg
  EXA_MINB=$1 EXA_SC_SLOW_INLINE=$2 timeout 300 python tools/set_timing.py mp96_case1354 set >> $OUT 2>> gpurun_out/${T}_regs.err
done
for cfg in "4 0" "4 1" "3 1"; do
  set -- $cfg
  EXA_MINB=$1 EXA_SC_SLOW_INLINE=$2 timeout 600 python tools/set_timing.py n1_case2000 set >> $OUT 2>> gpurun_out/${T}_regs.err
done
echo done
