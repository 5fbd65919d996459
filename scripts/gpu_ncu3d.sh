cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KR:-k3_central|k3_cwenoz|k3_muscl}" -s ${S:-3} -c ${C:-3} -o gpurun_out/${NAME:-p3d} python scripts/prof3d.py --config ${CFG:-5} --n ${N:-64} --warmup 0 --steps 1 > gpurun_out/${NAME:-p3d}.log 2>&1; tail -2 gpurun_out/${NAME:-p3d}.log
