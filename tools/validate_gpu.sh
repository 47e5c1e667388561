#!/bin/bash
# Round validation (run under gpurun): GPU tests, smoke, bench (ours + reference arm), batched configs,
# ncu launch list + full capture of the set kernel (case13659) and of the N-1 set.
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload mp96_case1354 --cpu-seconds 5 > gpurun_out/${TAG}_bench_mp96.json 2> gpurun_out/${TAG}_bench_mp96.err
timeout 900 python bench.py --steps 3 --warmup 3 --sets-per-step 4 --workload n1_case2000 --no-cpu-baseline > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --sets-per-step 8 --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exa_k_set -s 24 -c 2 \
  -o gpurun_out/${TAG}_prof_set -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sets-per-step 8 \
  --e2e-steps 1 > gpurun_out/${TAG}_ncu_full_run.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:exa_k_set -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_n1 -f python tools/set_timing.py n1_case2000 set > gpurun_out/${TAG}_ncu_n1.log 2>&1
echo finished
