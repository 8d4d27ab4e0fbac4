# r01_p: checkpoint after the class-ordered ATOMIC layout: smoke, all GPU tests, default bench,
# reference arm, ATOMIC on every config, launch list, ncu --set full of k_atomic on cfg1/cfg4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "bench ref rc=$?" >> gpurun_out/rc.txt
for c in 0 1 2 3 4; do $B --config $c --variant atomic > gpurun_out/bench_c${c}_atomic.log 2>&1; echo "bench c$c atomic rc=$?" >> gpurun_out/rc.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rc.txt
for c in 1 4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_atomic" -s 3 -c 1 -o gpurun_out/prof_c${c}_atomic python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant atomic > gpurun_out/ncu_c${c}_atomic.log 2>&1; echo "ncu c$c atomic rc=$?" >> gpurun_out/rc.txt
done
