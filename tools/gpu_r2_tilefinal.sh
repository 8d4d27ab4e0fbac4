# reduced final evidence after a TILE-only change: smoke, GPU tests, the default bench line, the
# reference arm, TILE on every config, ncu launch list and full captures of k_tile, TILE traces.
# (The other variants, the B5 sweep and the microbenchmarks are in the last gpu_r2_final.sh run.)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2tf}; mkdir -p $O
python -c "import bench; print(bench.source_hash())" > $O/src_hash.txt
nvidia-smi > $O/nvidia_smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "bench default rc=$?" >> $O/rc.txt
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_default.log 2>&1; echo "ref rc=$?" >> $O/rc.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30"
for c in 0 1 2 3 4; do
  $B --config $c --variant tile > $O/bench_c${c}_tile.log 2>&1; echo "bench c$c tile rc=$?" >> $O/rc.txt
done
for c in 2 4; do $B --config $c --variant tile --work 50 > $O/work50_c${c}_tile.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_default.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --per-config none > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
for cv in 4:tile 2:tile 3:tile 1:atomic 0:atomic 4:atomic; do c=${cv%%:*}; v=${cv##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_atomic" -s 3 -c 1 -o $O/prof_c${c}_$v python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --per-config none --variant $v > $O/ncu_c${c}_$v.log 2>&1; echo "ncu c$c $v rc=$?" >> $O/rc.txt
done
for c in 1 4; do timeout 300 python tools/tile_trace.py $c > $O/trace_c$c.txt 2>&1; done
