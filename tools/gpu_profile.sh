# Profiling pass on one GPU (via gpurun): per-op loop cycles, ncu launch list
# of the bench command, and ncu --set full captures of the top kernels.
mkdir -p gpurun_out
P=${PROFILE_TAG:-r1}
timeout 300 python tools/loop_profile.py > gpurun_out/loop_profile_$P.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_under_ncu_$P.log 2>&1
for K in ${NCU_KERNELS:-loop_jit k_gemm_tma ew_jit k_scan}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o gpurun_out/full_${P}_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${P}_$K.log 2>&1
done
ls -la gpurun_out
