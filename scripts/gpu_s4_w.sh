# session-4: p = 3 central kernel without the cp.async member prefetch, three blocks per SM (cpf0) vs prefetch, two blocks (base)
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do
  for v in base cpf0; do
    UCFVB_LIB=scratch/ab/$v.so timeout 600 python scripts/time_steps.py --config 3 --steps 40 --tag $v 2>&1 | tail -1 | cut -c1-200
  done
done
