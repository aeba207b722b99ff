mkdir -p gpurun_out
timeout 900 python tools/fw_debug.py fw_mlp_f32_I2B1024T8 fw_mlp_f32_I2B8T32 fw_ppo_f32_I1B1024T8E2M2 > gpurun_out/fw_debug.log 2>&1
timeout 900 python -m pytest -q tests/test_gpu_fullwidth.py tests/test_gpu_parity.py -k "fails_like or rng or ops_ or euclid or cumsum or divzero or ppo" > gpurun_out/pytest_sub.log 2>&1
tail -3 gpurun_out/pytest_sub.log; cat gpurun_out/fw_debug.log | cut -c1-400
