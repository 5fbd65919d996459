# A/B timing of two builds of libucfvb.so (scratch/ab/base.so vs new.so) on the 3D configs
cd "$GRAFT_REPO_ROOT"
for cfg in ${CFGS:-4 4c}; do
  for v in base new base new; do
    echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config $cfg --n ${N:-96} 2>&1 | tail -1 | cut -c1-150
  done
done
