cd $GRAFT_REPO_ROOT
O=gpurun_out/r2s3k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "forms_parity" > $O/pytest_forms.log 2>&1; echo "forms rc=$?" >> $O/rc.txt
B="python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 200"
for c in 0 1; do
  timeout 300 $B --config $c --variant atomic > $O/bench_c${c}_atomic.log 2>&1; echo "c$c rc=$?" >> $O/rc.txt
  for t in am5 am6; do (cd ab_$t && timeout 300 $B --config $c --variant atomic > ../$O/ab_${t}_c${c}.log 2>&1); echo "$t c$c rc=$?" >> $O/rc.txt; done
done
B="python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30"
timeout 300 $B --config 4 --variant atomic > $O/bench_c4_atomic.log 2>&1
for t in am5 am6; do (cd ab_$t && timeout 300 $B --config 4 --variant atomic > ../$O/ab_${t}_c4.log 2>&1); done
