# ncu --set full of the C3 learner's thin kernels (raw CSV exports only)
mkdir -p gpurun_out
P=${PROFILE_TAG:-r2e}
for K in 'k_thin_smallv<float, .int.4, .bool.1, .int.4>:smallv_gate' 'k_thin_contract<float, .int.16, .bool.1>:contract' 'k_thin_rows<float, .int.8, .int.2>:rows'; do
  RX=${K%%:*}; NM=${K##*:}
  timeout 900 ncu --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k "regex:$RX" -c 1 \
    -o gpurun_out/full_${P}_c3_$NM python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${P}_c3_$NM.log 2>&1
  ncu -i gpurun_out/full_${P}_c3_$NM.ncu-rep --page raw --csv > gpurun_out/full_${P}_c3_${NM}_raw.csv 2>/dev/null
  ncu -i gpurun_out/full_${P}_c3_$NM.ncu-rep --page source --csv > gpurun_out/full_${P}_c3_${NM}_src.csv 2>/dev/null
  rm -f gpurun_out/full_${P}_c3_$NM.ncu-rep
done
ls -la gpurun_out/full_${P}_*
