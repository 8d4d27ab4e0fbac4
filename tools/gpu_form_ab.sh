# TILE form A/B in one tree via EES_TILE_FORM; parity of form 2 first
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/*
EES_TILE_FORM=2 timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not hybrid_color_full and not forms" > gpurun_out/pytest_form2.log 2>&1; echo "pytest form2 rc=$?" >> gpurun_out/rc.txt
EES_TILE_FORM=2 timeout 900 python -m pytest tests -m gpu -q -x -k "full_size and not hybrid" > gpurun_out/pytest_form2_full.log 2>&1; echo "pytest form2 full rc=$?" >> gpurun_out/rc.txt
for rep in 1 2; do for f in 1 2 0; do for c in 1 2 4 3; do
  EES_TILE_FORM=$f timeout 300 python bench.py --config $c --variant tile --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/form${f}_c${c}_r$rep.log 2>&1
done; done; done
