# session-4: register budgets of the lattice-class kernels: central with <= 136 registers (ce3), CWENOZ with two resident blocks (cw2)
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do
for v in base ce3 cw2; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
done
