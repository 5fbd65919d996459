# session-4: config-4 central with the phi ring (c3ring) against the default build (new)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/c3ring.so timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -3
for r in 1 2; do
for v in new c3ring; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 4 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
done
