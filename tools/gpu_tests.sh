# GPU test pass: the new parity tests first (fast feedback), then the whole suite.
mkdir -p gpurun_out
T=${TAG:-r2}
timeout 900 python -m pytest -q -x tests/test_gpu_fullwidth.py tests/test_gpu_parity.py -k "fullwidth or fails_like or rng or ops_ or euclid or cumsum or fw_" > gpurun_out/pytest_new_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new_$T.log
timeout 1800 python -m pytest -q tests -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
tail -3 gpurun_out/pytest_new_$T.log gpurun_out/pytest_gpu_$T.log
