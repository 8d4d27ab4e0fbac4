# ncu --set full capture of k_tile on the configs in NCU_CFGS (HEAD code), timings first
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2n}; mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30"
for c in ${NCU_CFGS:-4 3}; do
  timeout 300 $B --config $c --variant tile > $O/bench_c${c}_tile.log 2>&1; echo "bench c$c rc=$?" >> $O/rc.txt
  for t in ${AB_TREES}; do (cd ab_$t && timeout 300 $B --config $c --variant tile > ../$O/ab_${t}_c${c}.log 2>&1); echo "$t c$c rc=$?" >> $O/rc.txt; done
done
for c in ${NCU_CFGS:-4 3}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o $O/prof_c${c}_tile python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --per-config none --variant tile > $O/ncu_c${c}.log 2>&1; echo "ncu c$c rc=$?" >> $O/rc.txt
done
