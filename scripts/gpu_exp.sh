cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in 2 1 3; do timeout 600 python scripts/time_steps.py --config $cfg --steps 100 --tag "divrn-int" 2>&1 | tail -1; done
PROF_NAME=prof_r1j PROF_KERNELS="k_troubled_split|k_central_tma" PROF_SKIP=4 PROF_COUNT=2 bash scripts/gpu_prof.sh > /dev/null 2>&1
