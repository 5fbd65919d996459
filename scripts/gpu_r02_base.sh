# round-2 baseline: config 3 timing + ncu --set full of the central and troubled kernels
cd "$GRAFT_REPO_ROOT"
timeout 900 python scripts/time_steps.py --config 3 --steps 20 --tag base 2>&1 | tail -1 | tee gpurun_out/r02_base_time.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_split|k_central_tma|k_face_flux|k_gather" -s 12 -c 4 -o gpurun_out/r02_base_c3 python scripts/prof_step.py --config 3 --warmup 1 --steps 1 > gpurun_out/r02_base_ncu.log 2>&1
tail -3 gpurun_out/r02_base_ncu.log
