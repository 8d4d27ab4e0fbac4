cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
timeout 300 python tools/diag_floor.py > gpurun_out/diag_floor.txt 2>&1
for tree in ab_u2 .; do for c in 0 1 2 3 4; do
  (cd $tree && timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 30) > gpurun_out/ab_$(basename $tree)_c$c.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not hybrid_color_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
