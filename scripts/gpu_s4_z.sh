# session-4: lattice central kernel with the gather in two halves, four resident blocks (half) vs three (base), config 5
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/half.so timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -2
for v in base half base half; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
