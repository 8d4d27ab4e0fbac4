# A/B: same bench in several trees (with a parity spot-check in each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
for tree in ab_a ab_b ab_v8 .; do
  (cd $tree && timeout 600 python -m pytest tests -m gpu -q -x -k "parity_reduced and tile" > ../gpurun_out/ab_$(basename $tree)_pytest.log 2>&1)
  for c in 3 2 4 1; do
  (cd $tree && timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 30) > gpurun_out/ab_$(basename $tree)_c$c.log 2>&1
done; done
