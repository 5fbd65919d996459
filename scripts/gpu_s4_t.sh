# session-4: lane-per-point flux kernels with eight resident blocks (f3b8, 64 registers) vs unbounded (base, 72)
cd "$GRAFT_REPO_ROOT"
for cfg in 5 4; do
for v in base f3b8 base f3b8; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config $cfg --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
done
