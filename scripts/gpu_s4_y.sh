# session-4: p = 3 central kernel, four resident blocks with only pinv and phi staged (c4) vs three blocks (base, no member prefetch)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/c4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  for v in base c4; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
