# round-1 (session 3) full check: smoke, gpu tests, default bench, per-config x variant, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
for c in 0 1 2 3 4; do for v in atomic gather tile color; do
  if [ "$v" = color ] && [ $c = 2 -o $c = 4 ]; then continue; fi
  timeout 300 python bench.py --config $c --variant $v --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_$v.log 2>&1; echo "bench c$c $v rc=$?" >> gpurun_out/rc.txt
done; done
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rc.txt
for c in 1 3 4; do for v in atomic tile; do
B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant $v"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_atomic|k_tile" -s 3 -c 1 -o gpurun_out/prof_c${c}_$v $B > gpurun_out/ncu_c${c}_$v.log 2>&1; echo "ncu c$c $v rc=$?" >> gpurun_out/rc.txt
done; done
