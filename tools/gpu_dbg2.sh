mkdir -p gpurun_out
timeout 600 python tools/tc_bias.py > gpurun_out/tc_bias.log 2>&1
timeout 1800 python -m pytest -q tests -m gpu > gpurun_out/pytest_gpu_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2b.log
cat gpurun_out/tc_bias.log; grep -E "^FAILED|passed|failed" gpurun_out/pytest_gpu_r2b.log | tail -20
