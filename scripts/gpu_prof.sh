set -x
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_step.py --steps 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${PROF_KERNELS:-k_flux|k_troubled}" -s ${PROF_SKIP:-8} -c ${PROF_COUNT:-2} -o gpurun_out/${PROF_NAME:-prof} python scripts/prof_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
