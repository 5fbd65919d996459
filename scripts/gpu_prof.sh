set -x
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_step.py --steps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -s 48 -c 16 --csv --log-file gpurun_out/launches.csv python scripts/prof_step.py --steps 1 > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cwenoz|k_central|k_flux" -s 12 -c 3 -o gpurun_out/prof_r1 python scripts/prof_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out
