# session-4: full suite on the current tree (CN=1, 3D batch call) + 3D bench lines
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for cfg in 4 5; do
  timeout 1500 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/s4i_bench_$cfg.json 2> gpurun_out/s4i_bench_$cfg.err; echo bench$cfg=$?
done
