cd $GRAFT_REPO_ROOT; O=gpurun_out/r2t5; mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e --per-config none --steps 30 --variant tile"
timeout 400 $B --config 3 > $O/c3_f0.log 2>&1; echo "f0 rc=$?" >> $O/rc.txt
timeout 400 $B --config 3 --tile-form 1 > $O/c3_f1.log 2>&1; echo "f1 rc=$?" >> $O/rc.txt
timeout 400 $B --config 4 --tile-form 0 > $O/c4_f0.log 2>&1; echo "c4 f0 rc=$?" >> $O/rc.txt
