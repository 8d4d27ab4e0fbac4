# round 2: baseline timing + ncu full captures of k_tile on cfg2/cfg3/cfg4 (HEAD code)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
O=gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
for c in 2 3 4; do
  timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c${c}_tile.log 2>&1; echo "bench c$c rc=$?" >> $O/rc.txt
done
for c in 4 2 3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o $O/prof_c${c}_tile python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant tile > $O/ncu_c${c}.log 2>&1; echo "ncu c$c rc=$?" >> $O/rc.txt
done
