# final: smoke, all GPU tests, default bench x3 (AUTO choice stability)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for r in 1 2 3; do timeout 300 python bench.py > gpurun_out/bench_default_r$r.log 2>&1; echo "bench r$r rc=$?" >> gpurun_out/rc.txt; done
for c in 0 2 3 4; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_auto.log 2>&1; done
