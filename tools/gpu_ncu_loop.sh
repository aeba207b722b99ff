mkdir -p gpurun_out
T=${TAG:-r2g}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_mlp -c 1 \
  -o gpurun_out/full_${T}_loop_mlp python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_loop_$T.log 2>&1
tail -3 gpurun_out/ncu_loop_$T.log
