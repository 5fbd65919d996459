# session-4: div_rn + slot-line prefetch in the coop stores + packed-lane flux (new) against base, config 5; launch list
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -3
for v in base new base new; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
echo -n "new "; timeout 600 python scripts/prof3d.py --config 4c --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/s4_launches_5.csv python scripts/prof3d.py --config 5 --warmup 1 --steps 1 > gpurun_out/s4_ncu_launch5.log 2>&1; tail -1 gpurun_out/s4_ncu_launch5.log
