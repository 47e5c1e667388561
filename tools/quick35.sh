#!/bin/bash
TAG=${1:-q35}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { w=$1; shift; env "$@" timeout 300 python tools/set_timing.py $w set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run case13659
run case13659 EXA_GROUP_MAX=4
run case13659 EXA_GROUP_MAX=4 EXA_SEG_FILTER=heavy
run case13659 EXA_ATTACH_AUGS=0
run mp96_case1354
run mp96_case1354 EXA_GROUP_MAX=4
run n1_case2000
run n1_case2000 EXA_GROUP_MAX=4
echo done
