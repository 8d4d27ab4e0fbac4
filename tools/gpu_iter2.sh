# iteration: gpu tests (quick), tile+atomic bench on all configs, ncu of chosen (config, variant)
# usage: bash tools/gpu_iter2.sh "<cfg:variant ...>"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -rf gpurun_out/*
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -k "not full_size and not hybrid_color_full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
for c in 1 0 2 3 4; do for v in tile atomic; do
  timeout 300 python bench.py --config $c --variant $v --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/bench_c${c}_$v.log 2>&1; echo "bench c$c $v rc=$?" >> gpurun_out/rc.txt
done; done
for cv in ${1:-1:tile}; do c=${cv%%:*}; v=${cv##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_atomic" -s 3 -c 1 -o gpurun_out/prof_c${c}_$v python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --variant $v > gpurun_out/ncu_c${c}_$v.log 2>&1; echo "ncu c$c $v rc=$?" >> gpurun_out/rc.txt
done
