# session-4: DMMA smem strides + transposed gather (new) against the side-major build (base) on config 5;
# next-tile L2 prefetch in the per-cell troubled kernel (pfd) against cur on config 3
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -3
for cfg in 5; do
  for v in base new base new; do
    echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config $cfg --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
  done
done
for r in 1 2; do
  for v in cur pfd; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_cwenoz|k3_muscl" -s 3 -c 3 -o gpurun_out/s4b_p3d_5 python scripts/prof3d.py --config 5 --n 64 --warmup 0 --steps 1 > gpurun_out/s4b_ncu3d_5.log 2>&1; tail -2 gpurun_out/s4b_ncu3d_5.log
