# round 2: 3D + decomposition tests, then bench lines of every config (profiles/r02_bench_<cfg>.json)
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_3d.py tests/test_gpu_decompose.py -q -x 2>&1 | tail -1
for cfg in 1 2; do
  timeout 900 python bench.py --config $cfg --steps 50 --warmup 5 > gpurun_out/r02_bench_$cfg.log 2>&1; tail -1 gpurun_out/r02_bench_$cfg.log | cut -c1-300
done
for cfg in 4 4c 5; do
  timeout 1500 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/r02_bench_$cfg.log 2>&1; tail -1 gpurun_out/r02_bench_$cfg.log | cut -c1-300
done
