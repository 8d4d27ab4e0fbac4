# r01_n: ncu source-level capture of k_tile on cfg2 and cfg4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
for c in 2 4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 3 -c 1 -o gpurun_out/prof_c${c}_tile python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant tile > gpurun_out/ncu_c${c}.log 2>&1; echo "ncu c$c rc=$?" >> gpurun_out/rc.txt
done
