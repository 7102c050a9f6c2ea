#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for SG in 1184 296 148 74; do
  IPM_SIDE_GRID=$SG PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/side_grid.jsonl 2>&1
done
timeout 300 ./scripts/micro/stream_bw > $OUT/stream_bw.jsonl 2>&1
