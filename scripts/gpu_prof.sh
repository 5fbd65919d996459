set -x
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_step.py --steps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -s ${LAUNCH_SKIP:-52} -c ${LAUNCH_COUNT:-16} --csv --log-file gpurun_out/launches.csv python scripts/prof_step.py --steps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${PROF_KERNELS:-k_central_tma|k_troubled_tma|k_troubled_split|k_face_flux|k_gather_rk}" -s ${PROF_SKIP:-12} -c ${PROF_COUNT:-4} -o gpurun_out/${PROF_NAME:-prof} python scripts/prof_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
