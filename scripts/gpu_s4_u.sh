# session-4: flux kernels with ten resident blocks (f3b10) vs eight (base); 3D tests on base
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -2
for v in base f3b10 base f3b10; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
