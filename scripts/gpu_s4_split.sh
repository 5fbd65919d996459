# session-4: CWENOZ and MUSCL tiles of the per-cell troubled kernel in two launches (split) vs one (base)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/split.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py tests/test_gpu_run.py tests/test_gpu_decompose.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  for v in base split; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
