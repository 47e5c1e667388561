free -g | head -2; nproc; nvidia-smi -L
timeout 1800 python tools/parity_report.py --out gpurun_out/parity_r02.json > gpurun_out/parity_r02.log 2>&1
echo "rc=$?" >> gpurun_out/parity_r02.log
EXA_EXACT_ZERO_SIGN=1 timeout 1800 python tools/parity_report.py --out gpurun_out/parity_r02_exact.json > gpurun_out/parity_r02_exact.log 2>&1
echo "rc=$?" >> gpurun_out/parity_r02_exact.log
tail -3 gpurun_out/parity_r02.log gpurun_out/parity_r02_exact.log
