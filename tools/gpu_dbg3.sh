mkdir -p gpurun_out
timeout 600 python tools/tc_bias.py > gpurun_out/tc_bias2.log 2>&1
timeout 900 python tools/fw_debug.py fw_mlp_f32_I2B1024T8 > gpurun_out/fw_debug2.log 2>&1
timeout 900 python -m pytest -q tests/test_gpu_kernels.py > gpurun_out/pytest_kern.log 2>&1
cat gpurun_out/tc_bias2.log; cut -c1-300 gpurun_out/fw_debug2.log; tail -3 gpurun_out/pytest_kern.log
