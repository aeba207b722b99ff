mkdir -p gpurun_out
T=${TAG:-r2f}
timeout 300 python tools/loop_profile.py c2 > gpurun_out/loop_profile_$T.txt 2>&1
cat gpurun_out/loop_profile_$T.txt | head -20
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "loop" > gpurun_out/pytest_loop_$T.log 2>&1; tail -2 gpurun_out/pytest_loop_$T.log
timeout 600 python -m pytest -q tests/test_gpu_backend.py > gpurun_out/pytest_backend_$T.log 2>&1; grep -E "^E |Error|passed|failed" gpurun_out/pytest_backend_$T.log | head -20
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_$T.json 2> gpurun_out/bench_c2_$T.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_$T.json').read().strip().splitlines()[-1])
print('c2', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['value']/1e6,2), d['breakdown']['family_ms_per_step'])
"
