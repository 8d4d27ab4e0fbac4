# round 2 final evidence: smoke, GPU tests, the default bench line (driver shape), the reference
# arm, every config x variant, B5 sweep, FP64 work mode, NEXT-3 adder, microbenchmarks, ncu launch
# list and full captures, TILE traces.  Everything lands in gpurun_out/$R2TAG.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2final}; mkdir -p $O
python -c "import bench; print(bench.source_hash())" > $O/src_hash.txt
nvidia-smi > $O/nvidia_smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default_s20.log 2>&1; echo "bench default s20 rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "bench default rc=$?" >> $O/rc.txt
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_default.log 2>&1; echo "ref rc=$?" >> $O/rc.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30"
for c in 0 1 2 3 4; do for v in atomic gather tile color color_buf; do
  $B --config $c --variant $v > $O/bench_c${c}_$v.log 2>&1; echo "bench c$c $v rc=$?" >> $O/rc.txt
done
  $B --config $c --variant color --rule hybrid > $O/bench_c${c}_colorh64.log 2>&1
done
for c in 2 4; do for v in tile atomic; do $B --config $c --variant $v --work 50 > $O/work50_c${c}_$v.log 2>&1; done; done
for n in adder64 adder64_r14 adder64_r89; do
  for v in atomic tile; do $B --netlist $n --variant $v > $O/bench_${n}_$v.log 2>&1; done
  $B --netlist $n --variant color --rule paper --steps 10 > $O/bench_${n}_colorpaper.log 2>&1
done
python -c "
from paper_2604_03079_b200 import fp64_peak, red_throughput
print('fp64_peak_tflops', fp64_peak()); print('red_spread_gops', red_throughput(0)); print('red_same_addr_gops', red_throughput(1))" > $O/microbench.txt 2>&1
timeout 1800 python bench.py --sweep --steps 10 --sweep-out $O/sweep_b5.jsonl > $O/sweep.log 2>&1; echo "sweep rc=$?" >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_default.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --per-config none > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
for cv in 4:tile 2:tile 3:tile 1:atomic 0:atomic 4:atomic; do c=${cv%%:*}; v=${cv##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_atomic" -s 3 -c 1 -o $O/prof_c${c}_$v python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --per-config none --variant $v > $O/ncu_c${c}_$v.log 2>&1; echo "ncu c$c $v rc=$?" >> $O/rc.txt
done
for c in 1 4; do timeout 300 python tools/tile_trace.py $c > $O/trace_c$c.txt 2>&1; done
