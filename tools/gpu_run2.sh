#!/bin/bash
# round-2 check: GPU tests, smoke, bench, zero-sign mode timings
T=${1:-r02a}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for w in case13659 mp96_case1354; do
  for z in 0 1; do EXA_EXACT_ZERO_SIGN=$z timeout 300 python tools/set_timing.py $w set >> gpurun_out/${T}_zs.jsonl 2>>gpurun_out/${T}_zs.err; done
done
tail -3 gpurun_out/${T}_gpu_tests.log
