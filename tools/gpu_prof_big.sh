cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --variant color --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bench_c${c}_color.log 2>&1; echo "bench c$c color rc=$?" >> gpurun_out/rc.txt
done
for c in 2 3 4; do for v in atomic tile gather; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant $v"
  timeout 300 $B > gpurun_out/plain_c${c}_$v.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_atomic|k_gather|k_tile" -s 3 -c 3 -o gpurun_out/prof_c${c}_$v $B > gpurun_out/ncu_c${c}_$v.log 2>&1; echo "ncu c$c $v rc=$?" >> gpurun_out/rc.txt
done; done
