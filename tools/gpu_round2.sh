mkdir -p gpurun_out
timeout 600 python bench_kernels.py > gpurun_out/bench_kernels.log 2>&1
timeout 600 python -m pytest tests/test_shard.py -m gpu -x -q > gpurun_out/pytest_shard.log 2>&1
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_gloo2.log 2>&1
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload c5 --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_gloo2.log 2>&1
cat gpurun_out/bench_kernels.log; tail -3 gpurun_out/pytest_shard.log; tail -c 1500 gpurun_out/bench_c2_gloo2.log; tail -c 1500 gpurun_out/bench_c5_gloo2.log
