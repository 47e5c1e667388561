#!/bin/bash
# compressed / objective kernels check + register-cap sweep
T=${1:-r02b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
bash tools/sweep_regs.sh $T
tail -3 gpurun_out/${T}_gpu_tests.log
