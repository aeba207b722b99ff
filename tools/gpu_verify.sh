# Round verification on one GPU: full gpu test suite, smoke, bench lines.
mkdir -p gpurun_out
P=${PROFILE_TAG:-r1d}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$P.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$P.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$P.log 2>&1
for W in c2 c3; do
  timeout 900 python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/bench_${W}_$P.json 2>gpurun_out/bench_${W}_$P.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$P.json 2>&1
tail -3 gpurun_out/pytest_gpu_$P.log
