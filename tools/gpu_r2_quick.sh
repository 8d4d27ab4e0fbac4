# quick check of a kernel change: GPU parity tests, TILE timing against the ab_head tree, trace
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R2TAG:-r2q}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.log 2>&1; echo "parity rc=$?" >> $O/rc.txt
B="python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30"
for c in ${MAIN_CFGS:-4 2}; do
  timeout 300 $B --config $c --variant tile > $O/bench_c${c}_tile.log 2>&1; echo "c$c rc=$?" >> $O/rc.txt
  for t in ${AB_TREES}; do (cd ab_$t && timeout 300 $B --config $c --variant tile > ../$O/ab_${t}_c${c}.log 2>&1); echo "$t c$c rc=$?" >> $O/rc.txt; done
done
timeout 300 python tools/tile_trace.py 4 > $O/trace_c4.txt 2>&1
