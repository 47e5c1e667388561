#!/bin/bash
# GPU tests, bench (ours + reference arm), host info.
TAG=${1:-r}
mkdir -p gpurun_out
(nproc; lscpu | head -20; nvidia-smi) > gpurun_out/${TAG}_host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
echo done
