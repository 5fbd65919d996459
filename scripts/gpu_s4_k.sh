# session-4: batched div_rn range tests in k_troubled_cells (divb vs base), configs 3 and 2 (lists)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/divb.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2 3; do
  for v in base divb; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
for v in base divb; do
  UCFVB_LIB=scratch/ab/$v.so UCFVB_TROUBLED=lists timeout 600 python scripts/time_steps.py --config 2 --steps 200 --tag $v-lists 2>&1 | tail -1 | cut -c1-200
done
