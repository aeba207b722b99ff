# Round-2 evidence on one GPU: full gpu tests + smoke, bench lines (C2 default,
# C3, C4, reference arm), ncu launch lists (C2, C3), ncu --set full of the top
# kernels, kernel roofline bench.
mkdir -p gpurun_out
P=${PROFILE_TAG:-r2h}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$P.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$P.log
tail -3 gpurun_out/pytest_gpu_$P.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$P.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default_$P.json 2> gpurun_out/bench_default_$P.err
for W in c3 c4; do
  timeout 1200 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$P.json 2>gpurun_out/bench_${W}_$P.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$P.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/launches_$P.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_under_ncu_$P.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/launches_c3_$P.csv python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_c3_under_ncu_$P.log 2>&1
for K in ${NCU_KERNELS:-loop_mlp k_gemm_tmap k_thin_small k_thin_contract_bulk}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o gpurun_out/full_${P}_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_${P}_$K.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tmap -c 1 \
  -o gpurun_out/full_${P}_c3_gemm python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_full_${P}_c3_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_thin_smallv -c 1 \
  -o gpurun_out/full_${P}_c3_smallv python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_full_${P}_c3_smallv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:smallv<float, .int.4, .bool.1, .int.4>" -c 1 \
  -o gpurun_out/full_${P}_c3_sumgate python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_full_${P}_c3_sumgate.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tma -c 1 \
  -o gpurun_out/full_${P}_k_scan_tma python bench_kernels.py --only returns_bt --reps 1 \
  > gpurun_out/ncu_full_${P}_k_scan_tma.log 2>&1
timeout 600 python bench_kernels.py > gpurun_out/bench_kernels_$P.jsonl 2>&1
# keep the copy-back under 64 MiB: raw-page CSV exports instead of the reports,
# a per-kernel summary instead of the C3 launch list
for f in gpurun_out/full_${P}_*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null && rm -f "$f"
done
python tools/launch_summary.py gpurun_out/launches_$P.csv gpurun_out/launches_c3_$P.csv > gpurun_out/launches_summary_$P.txt 2>&1
rm -f gpurun_out/launches_c3_$P.csv gpurun_out/loop_src_*.cu
du -sh gpurun_out
timeout 300 python tools/loop_profile.py c2 > gpurun_out/loop_profile_$P.txt 2>&1
for f in gpurun_out/bench_*_$P.json; do echo "$f"; tail -c 400 "$f"; echo; done
