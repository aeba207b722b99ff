mkdir -p gpurun_out
T=${TAG:-r2d}
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "loop or jit" > gpurun_out/pytest_loop_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop_$T.log
tail -3 gpurun_out/pytest_loop_$T.log
timeout 900 python -m pytest -q tests/test_gpu_fullwidth.py > gpurun_out/pytest_fw_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fw_$T.log
tail -3 gpurun_out/pytest_fw_$T.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_$T.json 2> gpurun_out/bench_c2_$T.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_$T.json').read().strip().splitlines()[-1])
print('c2', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['value']/1e6,2), d['breakdown']['family_ms_per_step'])
"
tail -3 gpurun_out/bench_c2_$T.err
