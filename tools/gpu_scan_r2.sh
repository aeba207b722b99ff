# TMA scan: parity tests, then a stage sweep at E=32768, T=1000
mkdir -p gpurun_out
T=${TAG:-r2s}
timeout 900 python -m pytest -q tests/test_gpu_kernels.py -m gpu -k "scan or gae" -x > gpurun_out/pytest_scan_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scan_$T.log
tail -15 gpurun_out/pytest_scan_$T.log
for ns in auto 2 3 4 6 8; do
  if [ "$ns" = auto ]; then unset RTB200_SCAN_STAGES; else export RTB200_SCAN_STAGES=$ns; fi
  echo "stages $ns"
  for k in returns_bt gae_bt; do timeout 300 python bench_kernels.py --only $k 2>&1 | tail -1 | cut -c1-200; done
done
unset RTB200_SCAN_STAGES
timeout 300 python bench_kernels.py --only returns_tb 2>&1 | tail -1 | cut -c1-200
