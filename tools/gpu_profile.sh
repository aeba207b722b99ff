# Profiling pass on one GPU (via gpurun): per-op loop cycles, ncu launch list
# of the bench command, ncu --set full captures of the top kernels, kernel
# roofline bench and the bench lines of every workload.
mkdir -p gpurun_out
P=${PROFILE_TAG:-r1}
timeout 300 python tools/loop_profile.py c2 > gpurun_out/loop_profile_$P.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_under_ncu_$P.log 2>&1
for K in ${NCU_KERNELS:-loop_jit k_gemm_tma ew_jit k_thin}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o gpurun_out/full_${P}_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${P}_$K.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -c 1 \
  -o gpurun_out/full_${P}_k_scan_pipe python bench_kernels.py --only returns_bt --reps 1 \
  > gpurun_out/ncu_full_${P}_k_scan.log 2>&1
timeout 600 python bench_kernels.py > gpurun_out/bench_kernels_$P.jsonl 2>&1
for W in c2 c3 c4; do
  timeout 1200 python bench.py --workload $W --steps 3 --warmup 3 > gpurun_out/bench_${W}_$P.json 2>&1
done
ls -la gpurun_out
