# TILE iteration: gpu tests, per-config tile + atomic bench, ncu of k_tile on cfg1/cfg4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt gpurun_out/*.log gpurun_out/*.ncu-rep
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for c in 1 0 2 3 4; do for v in tile atomic; do
  timeout 300 python bench.py --config $c --variant $v --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_$v.log 2>&1; echo "bench c$c $v rc=$?" >> gpurun_out/rc.txt
done; done
for c in ${NCU_CFGS:-1 4}; do
B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant tile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o gpurun_out/prof_c${c}_tile $B > gpurun_out/ncu_c${c}_tile.log 2>&1; echo "ncu c$c tile rc=$?" >> gpurun_out/rc.txt
done
