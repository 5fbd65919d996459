# A/B of 3D builds (scratch/ab/*.so) on configs 5, 4c and 4 (per-group us/stage)
cd "$GRAFT_REPO_ROOT"
[ -n "$TESTS" ] && UCFVB_LIB=scratch/ab/$TESTS.so timeout 900 python -m pytest tests/test_gpu_3d.py -q -x 2>&1 | tail -2
for cfg in ${CFGS:-5 4c 4}; do
  for v in ${LIBS:-base b3d cw3m3}; do
    echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/prof3d.py --config $cfg 2>&1 | tail -1 | cut -c1-170
  done
done
