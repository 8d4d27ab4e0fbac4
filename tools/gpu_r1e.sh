# new-feature check: COLOR_BUF, accept, work multiplier, fp64 peak; sweep with color_buf; FP64-bound bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -rf gpurun_out/*
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -k "not full_size and not hybrid_color_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20"
for c in 1 2 3 4; do
  $B --config $c --variant tile --work 50 > gpurun_out/work50_c${c}_tile.log 2>&1
  $B --config $c --variant atomic --work 50 > gpurun_out/work50_c${c}_atomic.log 2>&1
done
for c in 0 1 3; do $B --config $c --variant color_buf > gpurun_out/bench_c${c}_color_buf.log 2>&1; done
for c in 2 4; do $B --config $c --variant color_buf --rule hybrid > gpurun_out/bench_c${c}_color_buf_h.log 2>&1; done
for c in 1 2 3 4; do $B --config $c --variant gather > gpurun_out/bench_c${c}_gather_phases.log 2>&1; done
timeout 900 python bench.py --sweep --steps 10 --sweep-out gpurun_out/sweep_b5.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/rc.txt
