# iteration pass: gpu tests, C2/C3 bench lines, C3 per-record profile
mkdir -p gpurun_out
T=${TAG:-it}
timeout 1200 python -m pytest -q tests -m gpu -x > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
tail -4 gpurun_out/pytest_gpu_$T.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_$T.json 2> gpurun_out/bench_c2_$T.err
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$T.json 2> gpurun_out/bench_c3_$T.err
timeout 900 python tools/profile_records.py c3 40 > gpurun_out/records_c3_$T.txt 2>&1
python - <<PY
import json
for w in ("c2","c3"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{w}_$T.json").read().strip().splitlines()[-1])
        print(w, round(d["value"]/1e6,2), "M env-steps/s", round(d["ms_per_step"],3), "ms", "e2e", round(d["e2e"]["value"]/1e6,2), d["breakdown"]["family_ms_per_step"], d["roofline_step"]["frac"])
    except Exception as e: print(w, "ERR", e)
PY
head -25 gpurun_out/records_c3_$T.txt
timeout 300 python tools/loop_profile.py c2 > gpurun_out/loop_profile_$T.txt 2>&1; head -12 gpurun_out/loop_profile_$T.txt
