# session-4: MUSCL-only launch of the per-cell troubled kernel with 32 resident blocks (m32, 64 registers) vs 24 (base, 80)
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do
  for v in base m32; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
