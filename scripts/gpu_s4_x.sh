# session-4: p = 3 central kernel with three resident blocks: without the member prefetch (cpf0) or with it and a slim
# group B (pf3), vs two blocks (base); next-tile id-line prefetch in the lattice CWENOZ / MUSCL kernels (new vs base, config 5)
cd "$GRAFT_REPO_ROOT"
UCFVB_LIB=scratch/ab/pf3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py tests/test_gpu_run.py -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do
  for v in base cpf0 pf3; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
timeout 900 python -m pytest tests/test_gpu_3d.py -m gpu -q -x 2>&1 | tail -2
for v in base new base new; do
  echo -n "$v "; UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/prof3d.py --config 5 --warmup 2 --steps 3 2>&1 | tail -1 | cut -c1-220
done
