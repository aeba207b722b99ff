# Round evidence on one GPU: full gpu tests + smoke, bench lines (C2 default,
# C3, C4, reference arm), ncu launch list of the default bench, ncu --set full
# of the top kernels, kernel roofline bench, loop per-op cycles.
mkdir -p gpurun_out
P=${PROFILE_TAG:-r1d}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$P.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$P.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$P.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default_$P.json 2> gpurun_out/bench_default_$P.err
for W in c3 c4; do
  timeout 1200 python bench.py --workload $W --steps 3 --warmup 3 > gpurun_out/bench_${W}_$P.json 2>gpurun_out/bench_${W}_$P.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$P.json 2>&1
timeout 300 python tools/loop_profile.py c2 > gpurun_out/loop_profile_$P.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_under_ncu_$P.log 2>&1
for K in ${NCU_KERNELS:-loop_jit k_gemm_tma ew_jit k_thin}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o gpurun_out/full_${P}_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${P}_$K.log 2>&1
done
timeout 600 python bench_kernels.py > gpurun_out/bench_kernels_$P.jsonl 2>&1
tail -2 gpurun_out/pytest_gpu_$P.log
# multi-rank functional check of the bench's sharded path (2 gloo ranks on one GPU)
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_gloo2_$P.log 2>&1
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload c5 --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_gloo2_$P.log 2>&1
