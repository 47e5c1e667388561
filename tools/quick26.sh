#!/bin/bash
TAG=${1:-q26}
mkdir -p gpurun_out
EXA_TRACE=1 EXA_PDL=0 timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace.npz > gpurun_out/${TAG}.log 2>&1
EXA_TRACE=1 EXA_PDL=0 EXA_SEG_FILTER=heavy timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace_heavy.npz >> gpurun_out/${TAG}.log 2>&1
EXA_TRACE=1 EXA_PDL=0 timeout 300 python tools/trace_set.py case2000 gpurun_out/${TAG}_trace_2000.npz >> gpurun_out/${TAG}.log 2>&1
echo done
