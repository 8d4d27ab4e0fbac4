# round 2: TILE parity first, then timing (+ A/B trees ab_*) + ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2x}; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
if [ "${RUN_TESTS:-1}" = 1 ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
fi
if [ "${DEFAULT_BENCH:-0}" = 1 ]; then
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_default.log 2>&1; echo "bench default rc=$?" >> $O/rc.txt
fi
B="python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30"
for c in ${MAIN_CFGS:-4 2 3}; do
  timeout 300 $B --config $c --variant tile > $O/bench_c${c}_tile.log 2>&1; echo "bench c$c rc=$?" >> $O/rc.txt
  timeout 300 $B --config $c --variant atomic > $O/bench_c${c}_atomic.log 2>&1; echo "bench c$c atomic rc=$?" >> $O/rc.txt
done
for t in ${AB_TREES}; do
  for c in ${AB_CFGS:-4 2 3}; do (cd ab_$t && timeout 300 $B --config $c --variant tile > ../$O/ab_${t}_c${c}_tile.log 2>&1); echo "ab $t c$c rc=$?" >> $O/rc.txt; done
done
for c in ${NCU_CFGS:-4}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o $O/prof_c${c}_tile python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --per-config '' --variant tile > $O/ncu_c${c}.log 2>&1; echo "ncu c$c rc=$?" >> $O/rc.txt
done
