# session-4: lane-0 bulk-copy issue (l0) vs one copy per lane (new), config 3 and config 2 (lists)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/l0.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py tests/test_gpu_run.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  for v in new l0; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
for v in new l0; do
  UCFVB_LIB=scratch/ab/$v.so UCFVB_TROUBLED=lists timeout 600 python scripts/time_steps.py --config 2 --steps 200 --tag $v-lists 2>&1 | tail -1 | cut -c1-200
done
