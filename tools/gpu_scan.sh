mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -8
timeout 600 python bench_kernels.py 2>&1 | tee gpurun_out/bench_kernels.log
