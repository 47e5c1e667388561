#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload mp96_case1354 --cpu-seconds 5 > gpurun_out/${TAG}_bench_mp96.json 2> gpurun_out/${TAG}_bench_mp96.err
timeout 900 python bench.py --steps 3 --warmup 3 --sets-per-step 4 --workload n1_case2000 --no-cpu-baseline > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err
echo finished
