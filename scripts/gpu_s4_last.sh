# last check of the round: full GPU suite on the final library, bench lines of configs 1 and 2
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for cfg in 1 2; do
  timeout 900 python bench.py --config $cfg --steps 50 --warmup 5 > gpurun_out/s4_bench_$cfg.json 2> gpurun_out/s4_bench_$cfg.err; echo bench$cfg=$?
done
