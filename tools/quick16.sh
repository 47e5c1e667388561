#!/bin/bash
TAG=${1:-q16}
mkdir -p gpurun_out
EXA_TRACE=1 EXA_PERSIST=0 timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace_classic.npz > gpurun_out/${TAG}.log 2>&1
EXA_TRACE=1 EXA_PERSIST=4 timeout 300 python tools/trace_set.py case13659 gpurun_out/${TAG}_trace_p4.npz >> gpurun_out/${TAG}.log 2>&1
echo done
