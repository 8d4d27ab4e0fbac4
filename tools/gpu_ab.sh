# A/B: same bench in several trees (usage: bash tools/gpu_ab.sh "<trees>" "<configs>" <variant>)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
for tree in $1; do
  for c in $2; do
  (cd $tree && timeout 300 python bench.py --config $c --variant $3 --no-cpu-baseline --no-e2e --steps 30) > gpurun_out/ab_$(basename $tree)_c$c.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not hybrid_color_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
