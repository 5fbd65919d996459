set -x
cd "$GRAFT_REPO_ROOT"
for cfg in 4 4c 5; do timeout 600 python scripts/prof3d.py --config $cfg --n ${N:-96} > gpurun_out/prof3d_$cfg.log 2>&1; cat gpurun_out/prof3d_$cfg.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_cwenoz|k3_muscl|k3_face_flux" -s 8 -c 4 -o gpurun_out/p3d_4 python scripts/prof3d.py --config 4 --n 96 --warmup 0 --steps 1 > gpurun_out/ncu3d_4.log 2>&1; tail -3 gpurun_out/ncu3d_4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_cwenoz|k3_muscl" -s 6 -c 3 -o gpurun_out/p3d_5 python scripts/prof3d.py --config 5 --n 64 --warmup 0 --steps 1 > gpurun_out/ncu3d_5.log 2>&1; tail -3 gpurun_out/ncu3d_5.log
