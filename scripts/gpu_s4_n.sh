# session-4: 17 resident single-warp blocks (m17, <= 120 registers) vs 16 (new), config 3
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do
  for v in new m17; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
