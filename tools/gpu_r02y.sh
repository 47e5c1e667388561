#!/bin/bash
# host mirrors, take 2: spinning pool workers; host-function vs synchronous mirrors
T=${1:-r02y}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_threads.py -x -q -k "host or thread" -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -2 gpurun_out/${T}_tests.log
for cfg in "1 200 0" "1 0 0" "1 200 1" "0 200 0" "1 500 0"; do
  set -- $cfg
  EXA_HOST_MIRROR=$1 EXA_HOST_SPIN_US=$2 EXA_MIRROR_SYNC=$3 timeout 600 python bench.py --steps 10 --warmup 5 --no-extras --e2e-steps 8 > gpurun_out/${T}_$1_$2_$3.json 2> gpurun_out/${T}_$1_$2_$3.err
  python -c "import json; d=json.load(open('gpurun_out/${T}_$1_$2_$3.json')); e=d['e2e']; print('mirror $1 spin $2 sync $3:', round(e['value']), e['d2h_bytes_per_step'], 'seq', round(e['sequential_value']), 'np', round(e['numpy_api_value']), 'np_pinned', round(e['numpy_api_pinned_value']))"
done
