# session-4: 3D tests + 3D bench lines of the tree with five resident MUSCL blocks
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_run.py -m gpu -q -x 2>&1 | tail -2
for cfg in 5 4 4c; do
  timeout 1500 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/s4_bench_$cfg.json 2> gpurun_out/s4_bench_$cfg.err; echo bench$cfg=$?
done
