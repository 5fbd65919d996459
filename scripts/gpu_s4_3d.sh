# session-4 3D: side-major face points (new) against HEAD~ (base) on configs 5 / 4 / 4c, then ncu of config 5 and 4
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -3
for cfg in ${CFGS:-5 4 4c}; do
  for v in base new base new; do
    echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config $cfg --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_cwenoz|k3_muscl|k3_face_flux|k3_spread" -s 5 -c 5 -o gpurun_out/s4_p3d_5 python scripts/prof3d.py --config 5 --n 64 --warmup 0 --steps 1 > gpurun_out/s4_ncu3d_5.log 2>&1; tail -2 gpurun_out/s4_ncu3d_5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_face_flux" -s 2 -c 2 -o gpurun_out/s4_p3d_4 python scripts/prof3d.py --config 4 --n 96 --warmup 0 --steps 1 > gpurun_out/s4_ncu3d_4.log 2>&1; tail -2 gpurun_out/s4_ncu3d_4.log
