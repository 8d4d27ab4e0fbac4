# r01_m: bench with stream_ref, TILE traces of cfg2/cfg3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
for c in 2 4; do timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_tile.log 2>&1; done
for c in 2 3; do timeout 300 python tools/tile_trace.py $c > gpurun_out/trace_c$c.txt 2>&1; done
