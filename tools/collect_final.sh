#!/bin/bash
# gpurun_out/TAG (written by tools/gpu_r2_final.sh or gpu_r2_tilefinal.sh) -> profiles/TAG_*:
#   tools/collect_final.sh r02_g
set -e
cd "$(dirname "$0")/.."
T=$1; R=gpurun_out/$T
python tools/summarize.py $R profiles/${T}_final
cp $R/launches_default.csv profiles/${T}_launches_default.csv
cp $R/src_hash.txt profiles/${T}_src_hash.txt
for c in 1 4; do [ -f $R/trace_c$c.txt ] && cp $R/trace_c$c.txt profiles/${T}_trace_cfg$c.txt; done
[ -f $R/microbench.txt ] && cp $R/microbench.txt profiles/${T}_microbench.txt
if [ -f $R/sweep_b5.jsonl ]; then
  cp $R/sweep_b5.jsonl profiles/${T}_sweep_b5.jsonl
  python tools/sweep_md.py profiles/${T}_sweep_b5.jsonl $T > profiles/${T}_sweep_b5.md
fi
(echo "ref arm:"; grep '^{' $R/ref_default.log | cut -c1-600; echo; echo "pytest:"; tail -1 $R/pytest_gpu.log; echo "smoke:"; tail -1 $R/smoke.log; echo; echo "rc:"; tr '\n' ';' < $R/rc.txt; echo) > profiles/${T}_ref_tests.txt
(echo "# k_tile warp-stall attribution ($T captures)"; echo
 echo "From the source pages of the \`ncu --set full --import-source on\` captures (\`tools/ncu_stalls.py\`). The rows at \`BSSY\` / \`BRA\` with barrier stalls are the waits at B1 / B0; \`LDCU.64 … c[0x0][0x3f8]\` is the grid barrier."; echo
 for c in 4 2 3; do [ -f $R/prof_c${c}_tile.ncu-rep ] && python tools/ncu_stalls.py $R/prof_c${c}_tile.ncu-rep 12; done) > profiles/${T}_tile_stalls.md
echo "profiles/${T}_* written"
