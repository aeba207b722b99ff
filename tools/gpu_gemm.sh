mkdir -p gpurun_out
T=${TAG:-x}
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_fullwidth.py > gpurun_out/pytest_gemm_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_$T.log
grep -E "^E |passed|failed|rc=" gpurun_out/pytest_gemm_$T.log | head -20
timeout 600 python tools/tc_bias.py 2>&1 | grep "gemm=tma"
bash tools/gpu_bench_c2.sh
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$T.json 2> gpurun_out/bench_c3_$T.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c3_$T.json').read().strip().splitlines()[-1])
print('c3', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['value']/1e6,2), d['breakdown']['family_ms_per_step'])
"
