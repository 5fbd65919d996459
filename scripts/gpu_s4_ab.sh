# session-4 A/B: wide k_spread + 64-byte-line records (new) against HEAD (base), then the e2e pipeline
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for cfg in 3 2 1; do
  for r in 1 2; do
    for v in base new; do
      UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config $cfg --steps ${STEPS:-60} --tag $v 2>&1 | tail -1 | cut -c1-200
    done
  done
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s4_bench3_b.json 2> gpurun_out/s4_bench3_b.err; echo bench=$?
