# usage: bash tools/gpu_run.sh "<variants for ncu>"   (run under gpurun)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
NCUV=${1:-"tile atomic"}
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
for c in 0 1 2 3 4; do for v in atomic color gather tile; do
  if [ "$v" = color ] && [ $c = 2 -o $c = 4 ]; then continue; fi
  timeout 300 python bench.py --config $c --variant $v --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_$v.log 2>&1; echo "bench c$c $v rc=$?" >> gpurun_out/rc.txt
done; done
for v in $NCUV; do
  timeout 300 $B --variant $v > gpurun_out/plain_$v.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_atomic|k_gather|k_color|k_tile" -s 2 -c 2 -o gpurun_out/prof_$v $B --variant $v > gpurun_out/ncu_$v.log 2>&1; echo "ncu $v rc=$?" >> gpurun_out/rc.txt
done
