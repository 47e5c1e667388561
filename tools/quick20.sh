#!/bin/bash
TAG=${1:-q20}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_timing.jsonl; : > $OUT
run() { env "$@" timeout 300 python tools/set_timing.py case13659 set >> $OUT 2>> gpurun_out/${TAG}_timing.err; }
run EXA_PDL=0
run EXA_PDL=1
run EXA_PDL=0 EXA_SEG_FILTER=heavy
run EXA_PDL=0 EXA_SEG_FILTER=fold
run EXA_PDL=0 EXA_SEG_FILTER=light
run EXA_PDL=0 EXA_BUCKETS=0 EXA_ATTACH=0
run EXA_PDL=0 EXA_BUCKETS=0 EXA_ATTACH=0 EXA_SEG_FILTER=heavy
run EXA_PDL=0 EXA_BUCKETS=0 EXA_ATTACH=0 EXA_SEG_FILTER=fold
run EXA_PDL=0 EXA_BUCKETS=0 EXA_ATTACH=0 EXA_SEG_FILTER=light
run EXA_PDL=1 EXA_BUCKETS=0 EXA_ATTACH=0
echo done
