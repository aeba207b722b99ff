mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "blocked" 2>&1 | tail -4
timeout 1200 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
tail -c 3000 gpurun_out/bench_c4.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
