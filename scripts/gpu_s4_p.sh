# session-4: cell-major pinv + 16-byte shared loads in the fast-path central kernel (new) vs AoSoA (base)
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py tests/test_gpu_run.py tests/test_gpu_decompose.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  for v in base new; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
for cfg in 2 1; do
for v in base new base new; do
  UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config $cfg --steps 300 --tag $v 2>&1 | tail -1 | cut -c1-200
done
done
