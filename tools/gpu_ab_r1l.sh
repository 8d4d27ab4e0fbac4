# r01_l: ATOMIC grid A/B + streaming calibration
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
timeout 300 python tools/diag_floor.py > gpurun_out/floor.txt 2>&1; echo "floor rc=$?" >> gpurun_out/rc.txt
for rep in 1 2; do for tree in ab_head ab_grid; do for c in 0 1 2 3 4; do
  (cd $tree && timeout 300 python bench.py --config $c --variant atomic --no-cpu-baseline --no-e2e --steps 30) > gpurun_out/ab_${tree}_c${c}_r$rep.log 2>&1
done; done; done
