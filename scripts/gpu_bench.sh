cd "$GRAFT_REPO_ROOT"
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.log 2>&1; tail -1 gpurun_out/bench_torchrun.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
