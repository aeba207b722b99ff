# per-record step profiles (C2, C3), loop phase cycles, scan at 4x size, ncu of the TMA scan
mkdir -p gpurun_out
T=${TAG:-r2p}
timeout 600 python tools/profile_records.py c2 60 > gpurun_out/records_c2_$T.txt 2>&1
timeout 900 python tools/profile_records.py c3 80 > gpurun_out/records_c3_$T.txt 2>&1
timeout 300 python tools/loop_profile.py c2 > gpurun_out/loop_profile_$T.txt 2>&1
for k in returns_bt gae_bt; do timeout 300 python bench_kernels.py --only $k --envs 131072 2>&1 | tail -1 | cut -c1-200; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tma -c 1 \
  -o gpurun_out/full_${T}_k_scan_tma python bench_kernels.py --only returns_bt --reps 1 > gpurun_out/ncu_scan_$T.log 2>&1
tail -5 gpurun_out/loop_profile_$T.txt
