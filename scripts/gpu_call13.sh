#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python paper_2405_03584_b200/build.py --timeline >> $OUT/build.log 2>&1
for B in 1 0; do
  IPM_UPD_BIG=$B timeout 300 python scripts/timeline_probe.py C3 > $OUT/timeline_c3_big$B.log 2>&1
  IPM_UPD_BIG=$B PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/probe13.jsonl 2>&1
done
IPM_SYM_LDG=1 PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/probe13.jsonl 2>&1
IPM_SYM_LDG=1 timeout 300 python scripts/pcg_iter_probe.py C2 >> $OUT/probe13.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x > $OUT/pytest13.log 2>&1
IPM_SYM_LDG=1 timeout 600 python scripts/c5_probe.py 3 > $OUT/c5_ldg.jsonl 2>&1
