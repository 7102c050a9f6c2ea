#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python paper_2405_03584_b200/build.py --timeline >> $OUT/build.log 2>&1
for K in 1 0; do
  IPM_SPMV_KEEP=$K timeout 300 python scripts/timeline_probe.py C3 > $OUT/timeline_keep$K.log 2>&1
  IPM_SPMV_KEEP=$K PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/keep.jsonl 2>&1
done
for K in 1 0; do
  IPM_SPMV_KEEP=$K PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/keep.jsonl 2>&1
done
