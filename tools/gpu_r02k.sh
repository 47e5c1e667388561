#!/bin/bash
# full validation: GPU tests, smoke, bench (default), launch list
T=${1:-r02k}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 1 --sets-per-step 64 --no-extras --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/${T}_gpu_tests.log; cat gpurun_out/${T}_smoke.log
