#!/bin/bash
# in-place page locking of reused numpy buffers: GPU tests + the bench's numpy-API e2e legs
T=${1:-r02v2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hostpins.py tests/test_gpu_threads.py tests/test_gpu_consumers.py -x -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for reg in 1 0; do
  EXA_HOST_REGISTER=$reg timeout 600 python bench.py --steps 10 --warmup 5 --no-extras --e2e-steps 16 > gpurun_out/${T}_reg$reg.json 2> gpurun_out/${T}_reg$reg.err
  python -c "import json; d=json.load(open('gpurun_out/${T}_reg$reg.json')); e=d['e2e']; print('register $reg:', round(d['value']), 'e2e', round(e['value']), 'seq', round(e['sequential_value']), 'np', round(e['numpy_api_value']), 'np_pinned', round(e['numpy_api_pinned_value']))"
done
