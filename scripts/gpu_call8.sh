#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python paper_2405_03584_b200/build.py --timeline >> $OUT/build.log 2>&1
for SB in 256 128 64; do
  IPM_SIDE_BLOCK=$SB timeout 300 python scripts/timeline_probe.py C3 > $OUT/timeline_c3_sb$SB.log 2>&1
  IPM_SIDE_BLOCK=$SB PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/sideblock.jsonl 2>&1
done
