mkdir -p gpurun_out
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_gloo2.log 2>&1
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload c5 --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_gloo2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_trun1.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for f in gpurun_out/bench_c2_gloo2.log gpurun_out/bench_c5_gloo2.log gpurun_out/bench_c2_trun1.log gpurun_out/bench_ref.log; do echo "== $f"; tail -1 $f | cut -c1-400; done
nproc
