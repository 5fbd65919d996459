# session-4: three-group refill of the per-cell troubled kernel (b3on / b3cn vs b3off) on config 3 and 2;
# next-chunk id-line prefetch in the lattice central kernel (new vs nopfid) on config 5
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py tests/test_gpu_run.py tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -3
for r in 1 2; do
  for v in b3off b3on b3cn; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
for v in b3off b3on b3cn; do
  UCFVB_LIB=scratch/ab/$v.so UCFVB_TROUBLED=lists timeout 600 python scripts/time_steps.py --config 2 --steps 200 --tag $v-lists 2>&1 | tail -1 | cut -c1-200
done
for v in nopfid new nopfid new; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
