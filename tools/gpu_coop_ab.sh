# COLOR coop-form A/B (EES_COLOR_MODE forces the form)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -rf gpurun_out/coop_*
for tree in ab_head ab_c2 .; do for mode in coop launch; do for n in cfg1 cfg3 synth4000000_4 synth4000000_16; do
  (cd $tree && EES_COLOR_MODE=$mode timeout 300 python bench.py --netlist $n --variant color --no-cpu-baseline --no-e2e --steps 20) > gpurun_out/coop_$(basename $tree)_${mode}_$n.log 2>&1
done; done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "color_forms or parity_reduced or synth" > gpurun_out/pytest_coop.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_coop.txt
