#!/bin/bash
# A/B build tree: tools/ab_tree.sh NAME "-DFOO=1 -DBAR=2" -> ab_NAME/ (git-ignored) holding a
# copy of the package, netgen, oracle, bench.py and tests built with those defines.
set -e
cd "$(dirname "$0")/.."
name=$1; defs=$2
rm -rf ab_$name; mkdir -p ab_$name
cp -r paper_2604_03079_b200 netgen oracle include tests bench.py __graft_entry__.py ab_$name/
rm -rf ab_$name/paper_2604_03079_b200/build ab_$name/paper_2604_03079_b200/lib
cp MEASURED_PEAKS.json ab_$name/ 2>/dev/null || true
(cd ab_$name && EES_NVCC_DEFS="$defs" python -m paper_2604_03079_b200.build --force > /dev/null 2>&1 && python -c "import oracle; oracle.build()")
echo "built ab_$name ($defs)"
