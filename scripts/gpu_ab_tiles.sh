# A/B of k_troubled_cells tile sizes (scratch/ab/*.so) on config 3 and config 2 (per-cell lists)
cd "$GRAFT_REPO_ROOT"
export UCFVB_TROUBLED=lists
for r in 1 2; do
  for v in ${LIBS:-base nodskip tile8m16 tile16m8}; do
    UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/time_steps.py --config 3 --steps 10 --tag $v 2>&1 | tail -1 | cut -c1-130
  done
done
for v in ${LIBS:-base nodskip tile8m16 tile16m8}; do
  UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/time_steps.py --config 2 --steps 100 --tag $v 2>&1 | tail -1 | cut -c1-130
done
