# A/B of k_troubled_cells variants (scratch/ab/*.so) on config 3 (per-cell lists) and config 2
cd "$GRAFT_REPO_ROOT"
export UCFVB_TROUBLED=lists
for r in 1 2; do
  for v in ${LIBS:-base pf minb5 pfminb5}; do
    UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/time_steps.py --config 3 --steps 10 --tag $v 2>&1 | tail -1 | cut -c1-150
  done
done
for v in ${LIBS:-base pf minb5 pfminb5}; do
  UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/time_steps.py --config 2 --steps 100 --tag $v 2>&1 | tail -1 | cut -c1-150
done
