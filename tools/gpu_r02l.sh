#!/bin/bash
T=${1:-r02l}
mkdir -p gpurun_out
for ipt in 1 2 4; do
  EXA_CMP_IPT=$ipt timeout 600 python tools/compressed_timing.py case13659 >> gpurun_out/${T}_comp.jsonl 2>> gpurun_out/${T}_comp.err
done
timeout 300 python tools/set_timing.py case13659 set >> gpurun_out/${T}_set.jsonl 2>> gpurun_out/${T}_set.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 300 python tools/set_timing.py case13659 set >> gpurun_out/${T}_set.jsonl 2>> gpurun_out/${T}_set.err
cat gpurun_out/${T}_comp.jsonl gpurun_out/${T}_set.jsonl; head -c 300 gpurun_out/${T}_bench.json
