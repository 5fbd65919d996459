# 3D A/B: c3d (current: per-thread troubled stores, minBlocks 3 for staged p=3 CWENOZ) vs coop (cooperative
# troubled stores); config 4 central: cp.async (TMA off) vs TMA pinv+phi (c3d) vs TMA pinv only (tmapinv)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/coop.so timeout 900 python -m pytest tests/test_gpu_3d.py -q -x 2>&1 | tail -1
for cfg in 5 4c; do
  for v in base c3d coop; do
    echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/prof3d.py --config $cfg 2>&1 | tail -1 | cut -c1-170
  done
done
echo -n "c3d tma=0 "; UCFVB_CENTRAL3_TMA=0 UCFVB_LIB=scratch/ab/c3d.so timeout 900 python scripts/prof3d.py --config 4 2>&1 | tail -1 | cut -c1-170
echo -n "c3d tma=1 "; UCFVB_LIB=scratch/ab/c3d.so timeout 900 python scripts/prof3d.py --config 4 2>&1 | tail -1 | cut -c1-170
echo -n "tmapinv "; UCFVB_LIB=scratch/ab/tmapinv.so timeout 900 python scripts/prof3d.py --config 4 2>&1 | tail -1 | cut -c1-170
