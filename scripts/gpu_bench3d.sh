set -x
cd "$GRAFT_REPO_ROOT"
for cfg in ${CFGS:-4 4c 5}; do
  timeout 1200 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 3 > gpurun_out/bench3d_$cfg.log 2>&1; tail -1 gpurun_out/bench3d_$cfg.log
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:k3_ -s 16 -c 16 --csv --log-file gpurun_out/launches3d_5.csv python scripts/prof3d.py --config 5 --warmup 1 --steps 1 > gpurun_out/ncu_l5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:k3_ -s 16 -c 16 --csv --log-file gpurun_out/launches3d_4.csv python scripts/prof3d.py --config 4 --warmup 1 --steps 1 > gpurun_out/ncu_l4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_cwenoz|k3_muscl|k3_face_flux" -s 8 -c 4 -o gpurun_out/p3d_5f python scripts/prof3d.py --config 5 --warmup 0 --steps 1 > gpurun_out/ncu3d_5f.log 2>&1; tail -2 gpurun_out/ncu3d_5f.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_face_flux|k3_gather" -s 8 -c 3 -o gpurun_out/p3d_4f python scripts/prof3d.py --config 4 --warmup 0 --steps 1 > gpurun_out/ncu3d_4f.log 2>&1; tail -2 gpurun_out/ncu3d_4f.log
