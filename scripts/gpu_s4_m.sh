# session-4: ncu --set full of the trimmed k_troubled_cells (config 3)
cd "$GRAFT_REPO_ROOT"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_cells" -s 2 -c 1 -o gpurun_out/s4m_cells python scripts/prof_step.py --config 3 --warmup 1 --steps 1 > gpurun_out/s4m_cells.log 2>&1
tail -2 gpurun_out/s4m_cells.log
