# A/B timing of two builds of libucfvb.so (scratch/ab/base.so vs new.so) on the 2D configs
cd "$GRAFT_REPO_ROOT"
[ -n "$TESTS" ] && UCFVB_LIB=scratch/ab/new.so timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in ${CFGS:-2 1}; do
  for v in base new base new base new; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config $cfg --steps ${STEPS:-300} --tag $v 2>&1 | tail -1 | cut -c1-150
  done
done
