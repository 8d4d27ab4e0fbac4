# A/B of working tree (.) vs ab_head, TILE, + pytest subset: bash tools/gpu_ab4.sh "<configs>" <variant> [pytest-k]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
for rep in 1 2; do for tree in ab_head .; do for c in $1; do
  n=$( [ "$tree" = "." ] && echo new || echo head )
  (cd $tree && timeout 300 python bench.py --config $c --variant $2 --no-cpu-baseline --no-e2e --steps 30) > gpurun_out/ab_${n}_c${c}_r$rep.log 2>&1
done; done; done
if [ -n "$3" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$3" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt; fi
