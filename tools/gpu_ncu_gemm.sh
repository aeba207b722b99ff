mkdir -p gpurun_out
T=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tma -c 2 \
  -o gpurun_out/full_${T}_k_gemm_tma python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm_$T.log 2>&1
tail -2 gpurun_out/ncu_gemm_$T.log
