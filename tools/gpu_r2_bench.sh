# round 2: default bench line (driver-shaped) + the bench contract GPU tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.log 2>&1; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_bench.py -x -q > $O/pytest_bench.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
lscpu > $O/lscpu.txt 2>&1; cat /sys/fs/cgroup/cpu.max >> $O/lscpu.txt 2>&1; nproc >> $O/lscpu.txt
