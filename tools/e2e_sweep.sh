#!/bin/bash
# e2e sweep of D2H strategies
T=$1
for cfg in "dma 0" "dma 25000" "dma 100000" "store 0"; do
  set -- $cfg
  EXA_D2H=$1 EXA_D2H_GAP=$2 timeout 600 python bench.py --steps 10 --warmup 5 --no-extras --e2e-steps 6 > gpurun_out/${T}_$1_$2.json 2> gpurun_out/${T}_$1_$2.err
  python -c "import json; d=json.load(open('gpurun_out/${T}_$1_$2.json')); e=d['e2e']; print('$1 $2', round(e['value']), round(e['d2h_GBps'],1), round(e['sequential_value']), round(e['numpy_api_value']), round(e['numpy_api_pinned_value']))"
done
