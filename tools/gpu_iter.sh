# iteration: gpu tests, tile bench on all configs, traces, ncu of k_tile
# usage: bash tools/gpu_iter.sh "<ncu configs>" "<pytest -k expr>"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -rf gpurun_out/*
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -k "${2:-not nothing}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for c in 1 0 2 3 4; do
  timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_tile.log 2>&1; echo "bench c$c tile rc=$?" >> gpurun_out/rc.txt
done
for c in 1 4; do timeout 300 python tools/tile_trace.py $c > gpurun_out/trace_c$c.txt 2>&1; done
for c in ${1:-1 4}; do
B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant tile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o gpurun_out/prof_c${c}_tile $B > gpurun_out/ncu_c${c}_tile.log 2>&1; echo "ncu c$c tile rc=$?" >> gpurun_out/rc.txt
done
