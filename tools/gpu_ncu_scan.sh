mkdir -p gpurun_out
for K in returns_bt returns_tb; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -c 1 -o gpurun_out/scan_$K python bench_kernels.py --only $K --reps 1 > gpurun_out/ncu_scan_$K.log 2>&1
done
ls gpurun_out
