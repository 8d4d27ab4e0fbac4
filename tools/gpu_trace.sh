cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 1 3 4; do timeout 300 python tools/tile_trace.py $c > gpurun_out/trace_c$c.txt 2>&1; done
