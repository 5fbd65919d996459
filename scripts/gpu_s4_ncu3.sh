# ncu --set full of one stage of config 3 (six kernels per stage: central, spread, CWENOZ tiles, MUSCL tiles, flux, gather)
cd "$GRAFT_REPO_ROOT"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_cells|k_central_tma|k_face_flux|k_gather|k_spread" -s 12 -c 6 -o gpurun_out/s4_full3 python scripts/prof_step.py --config 3 --warmup 1 --steps 1 > gpurun_out/s4_ncu_full3.log 2>&1
tail -2 gpurun_out/s4_ncu_full3.log
