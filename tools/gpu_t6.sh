mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/loop_profile.py c2 2>&1 | grep -v Warn | head -14
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/bench_c2.log", "gpurun_out/bench_c3.log"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["breakdown"]["family_ms_per_step"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-3000:])
PY
