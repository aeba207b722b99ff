# Round-2 GPU pass: full GPU tests, smoke, C2/C3 bench lines.
mkdir -p gpurun_out
T=${TAG:-r2c}
timeout 1800 python -m pytest -q tests -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_$T.json 2> gpurun_out/bench_c2_$T.err
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$T.json 2> gpurun_out/bench_c3_$T.err
grep -E "^FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -15; tail -1 gpurun_out/smoke_$T.log
python - <<'PY'
import json
for w in ("c2","c3"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{w}_$T.json").read().strip().splitlines()[-1])
        print(w, round(d["value"]/1e6,2), "M env-steps/s", round(d["ms_per_step"],3), "ms", "e2e", round(d["e2e"]["value"]/1e6,2), d["breakdown"]["family_ms_per_step"])
    except Exception as e: print(w, "ERR", e)
PY
