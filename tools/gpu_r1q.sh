# round-1 checkpoint r01_q: smoke, full gpu tests, default bench, every config x variant, sweep, ncu, microbenchmarks
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -rf gpurun_out/*
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "bench ref rc=$?" >> gpurun_out/rc.txt
python -c "
from paper_2604_03079_b200 import fp64_peak, red_throughput
print('fp64_peak_tflops', fp64_peak()); print('red_spread_gops', red_throughput(0)); print('red_same_addr_gops', red_throughput(1))" > gpurun_out/microbench.txt 2>&1
for c in 0 1 2 3 4; do for v in atomic gather tile color color_buf; do
  if [ "$v" = color -o "$v" = color_buf ] && [ $c = 2 -o $c = 4 ]; then continue; fi
  $B --config $c --variant $v > gpurun_out/bench_c${c}_$v.log 2>&1; echo "bench c$c $v rc=$?" >> gpurun_out/rc.txt
done
  $B --config $c --variant color --rule hybrid > gpurun_out/bench_c${c}_colorh64.log 2>&1
  $B --config $c --variant color_buf --rule hybrid > gpurun_out/bench_c${c}_color_bufh64.log 2>&1
done
for c in 1 2 4; do for v in tile atomic; do $B --config $c --variant $v --work 50 > gpurun_out/work50_c${c}_$v.log 2>&1; done; done
for n in adder64 adder64_r14 adder64_r89; do
  for v in atomic tile; do $B --netlist $n --variant $v > gpurun_out/bench_${n}_$v.log 2>&1; done
  $B --netlist $n --variant color --rule paper --steps 10 > gpurun_out/bench_${n}_colorpaper.log 2>&1
done
timeout 1200 python bench.py --sweep --steps 10 --sweep-out gpurun_out/sweep_b5.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rc.txt
for cv in 1:atomic 1:tile 2:tile 3:tile 4:tile; do c=${cv%%:*}; v=${cv##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_atomic" -s 3 -c 1 -o gpurun_out/prof_c${c}_$v python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/ncu_c${c}_$v.log 2>&1; echo "ncu c$c $v rc=$?" >> gpurun_out/rc.txt
done
for c in 1 4; do timeout 300 python tools/tile_trace.py $c > gpurun_out/trace_c$c.txt 2>&1; done
