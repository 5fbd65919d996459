cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x 2>&1 | tail -1
for cfg in 2 1 3; do timeout 600 python scripts/time_steps.py --config $cfg --steps 100 --tag "gatherNT" 2>&1 | tail -1; done
sed -i 's/__global__ void __launch_bounds__(kBlock) k_face_flux(/__global__ void __launch_bounds__(kBlock, 10) k_face_flux(/' paper_2510_25906_b200/csrc/kernels.cuh
make -C paper_2510_25906_b200 -j8 > /dev/null 2>&1; grep -A3 "k_face_fluxILi2E" paper_2510_25906_b200/build/ptxas_solver.log | grep -E "registers|spill"
for cfg in 2 1; do timeout 600 python scripts/time_steps.py --config $cfg --steps 100 --tag "flux-lb10" 2>&1 | tail -1; done
