# A/B/n timing of several builds of libucfvb.so (scratch/ab/<name>.so) on the 2D configs.
#   LIBS="base new" CFGS="2 1" TESTLIB=new bash scripts/gpu_abn.sh
cd "$GRAFT_REPO_ROOT"
for t in $TESTLIB; do
  echo "tests with $t:"; UCFVB_LIB=scratch/ab/$t.so timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
done
for cfg in ${CFGS:-2}; do
  for r in 1 2 3; do
    for v in ${LIBS:-base new}; do
      UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config $cfg --steps ${STEPS:-300} --tag $v 2>&1 | tail -1 | cut -c1-150
    done
  done
done
