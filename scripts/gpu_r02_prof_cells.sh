# ncu --set full of k_troubled_cells (config 3 and config 2, per-cell lists) and k_spread
cd "$GRAFT_REPO_ROOT"
export UCFVB_TROUBLED=lists
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_cells|k_spread" -s 6 -c 2 -o gpurun_out/r02_cells_c3 python scripts/prof_step.py --config 3 --warmup 1 --steps 1 > gpurun_out/r02_cells_ncu3.log 2>&1
tail -2 gpurun_out/r02_cells_ncu3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_cells|k_troubled_split" -s 3 -c 1 -o gpurun_out/r02_cells_c2 python scripts/prof_step.py --config 2 --warmup 1 --steps 1 > gpurun_out/r02_cells_ncu2.log 2>&1
tail -2 gpurun_out/r02_cells_ncu2.log
