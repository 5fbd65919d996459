# session-4: micro-trims of k_troubled_cells (copy lanes' cell by shuffle, branch instead of per-store selects): new vs base
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py tests/test_gpu_run.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2 3; do
  for v in base new; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
