mkdir -p gpurun_out
T=${TAG:-x}
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_$T.json 2> gpurun_out/bench_c2_$T.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_c2_$T.json').read().strip().splitlines()[-1])
print('c2', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['value']/1e6,2), d['breakdown']['family_ms_per_step'])
for r in d['breakdown']['top']: print('   ', r)
"
