#!/bin/bash
# One gpurun session: GPU tests, bench, ncu launch list + full capture of the set kernel.
# usage: tools/gpu_run.sh TAG [skip_tests]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
if [ "$2" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
fi
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --sets-per-step 8 --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exa_k_set -s 24 -c 2 \
  -o gpurun_out/${TAG}_prof_set -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sets-per-step 8 \
  --e2e-steps 1 > gpurun_out/${TAG}_ncu_full_run.log 2>&1
echo finished
