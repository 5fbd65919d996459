# 3D A/B: round-1 store pattern (base) vs cooperative stores (c3d, c3dm3), TMA central on/off (config 4)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/c3d.so timeout 900 python -m pytest tests/test_gpu_3d.py -q -x 2>&1 | tail -2
for cfg in 5 4c; do
  for v in base c3d c3dm3; do
    echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/prof3d.py --config $cfg 2>&1 | tail -1 | cut -c1-170
  done
done
for t in 1 0; do
  echo -n "c3d central3_tma=$t "; UCFVB_CENTRAL3_TMA=$t UCFVB_LIB=scratch/ab/c3d.so timeout 900 python scripts/prof3d.py --config 4 2>&1 | tail -1 | cut -c1-170
done
