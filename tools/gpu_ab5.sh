# A/B of scratch trees: bash tools/gpu_ab5.sh "<trees>" "<configs>" <variant> [tree-for-pytest] [pytest-k]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
for rep in 1 2; do for tree in $1; do for c in $2; do
  (cd $tree && timeout 300 python bench.py --config $c --variant $3 --no-cpu-baseline --no-e2e --steps 30) > gpurun_out/ab_$(basename $tree)_c${c}_r$rep.log 2>&1
done; done; done
if [ -n "$4" ]; then (cd $4 && timeout 1500 python -m pytest tests -m gpu -q -x -k "$5") > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt; fi
