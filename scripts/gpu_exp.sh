cd "$GRAFT_REPO_ROOT"
bash scripts/gpu_bench.sh
PROF_NAME=prof_r1m bash scripts/gpu_prof.sh > /dev/null 2>&1
tail -2 gpurun_out/ncu_full.log
