# session-4: lattice-class MUSCL kernel with five resident blocks (m3b5, 72 registers) vs four (base), config 5
cd "$GRAFT_REPO_ROOT"
for v in base m3b5 base m3b5; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
