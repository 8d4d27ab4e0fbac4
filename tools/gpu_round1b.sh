cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
for v in atomic color gather; do timeout 300 python bench.py --variant $v --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.log 2>&1; echo "bench $v rc=$?" >> gpurun_out/rc.txt; done
for v in atomic gather color; do
  timeout 300 $B --variant $v > gpurun_out/plain_$v.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_atomic|k_gather|k_color" -s 3 -c 3 -o gpurun_out/prof_$v $B --variant $v > gpurun_out/ncu_$v.log 2>&1; echo "ncu $v rc=$?" >> gpurun_out/rc.txt
done
timeout 300 $B > gpurun_out/plain_default.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rc.txt
