#!/bin/bash
# host mirrors: host-path parity at scale + e2e with mirrors on/off and pool sizes
T=${1:-r02x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_threads.py -x -q -k "host or thread" -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for cfg in "1 8" "0 8" "1 4" "1 6" "1 12"; do
  set -- $cfg
  EXA_HOST_MIRROR=$1 EXA_HOST_FILL_THREADS=$2 timeout 600 python bench.py --steps 10 --warmup 5 --no-extras --e2e-steps 8 > gpurun_out/${T}_m$1_t$2.json 2> gpurun_out/${T}_m$1_t$2.err
  python -c "import json; d=json.load(open('gpurun_out/${T}_m$1_t$2.json')); e=d['e2e']; print('mirror $1 threads $2', round(e['value']), e['d2h_bytes_per_step'], round(e['sequential_value']), round(e['numpy_api_value']), round(e['numpy_api_pinned_value']))"
done
