mkdir -p gpurun_out
timeout 1200 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 1200 python bench.py --workload c4_noswap --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_noswap.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/bench_c4.log", "gpurun_out/bench_c4_noswap.log"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "peak", d["peak_hbm_bytes"]/1e9, d["peak_hbm_allocated_bytes"]/1e9, d.get("swap"))
        print("   ", d["breakdown"]["family_ms_per_step"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-3000:])
PY
