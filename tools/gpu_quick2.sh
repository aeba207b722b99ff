# Quick A/B on one GPU: loop parity tests, C2/C3 bench lines, loop per-op cycles.
# HYB_SWEEP="A=1,B=2 A=0": one loop_profile run per comma-separated env set.
mkdir -p gpurun_out
P=${PROFILE_TAG:-q}
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_$P.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$P.log
for W in ${WORKLOADS:-c2 c3}; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$P.json 2>gpurun_out/bench_${W}_$P.err
done
i=0
for V in ${HYB_SWEEP:-x}; do
  i=$((i+1))
  (for kv in $(echo "$V" | tr ',' ' '); do [ "$kv" = x ] || export "$kv"; done
   echo "env: $V"; timeout 300 python tools/loop_profile.py c2) > gpurun_out/loop_profile_${P}_$i.txt 2>&1
done
tail -2 gpurun_out/pytest_$P.log
