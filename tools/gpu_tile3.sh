cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt gpurun_out/*.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for c in 0 1 2 3 4; do
  timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_tile.log 2>&1; echo "bench c$c tile rc=$?" >> gpurun_out/rc.txt
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -k "full_size" > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest full rc=$?" >> gpurun_out/rc.txt
B="python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant tile"
timeout 300 $B > gpurun_out/plain_c1_tile.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o gpurun_out/prof_c1_tile3 $B > gpurun_out/ncu_c1_tile.log 2>&1; echo "ncu c1 tile rc=$?" >> gpurun_out/rc.txt
B="python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant tile"
timeout 300 $B > gpurun_out/plain_c3_tile.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o gpurun_out/prof_c3_tile3 $B > gpurun_out/ncu_c3_tile.log 2>&1; echo "ncu c3 tile rc=$?" >> gpurun_out/rc.txt
