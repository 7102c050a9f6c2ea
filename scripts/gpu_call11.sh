#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python paper_2405_03584_b200/build.py --timeline >> $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > $OUT/pytest_shard11.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu11.log 2>&1
timeout 300 python scripts/timeline_probe.py C3 > $OUT/timeline_c3_11.log 2>&1
for U in 1 2 4; do IPM_UNROLL=$U PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/unroll.jsonl 2>&1; done
for U in 1 2; do IPM_UNROLL=$U timeout 300 python scripts/pcg_iter_probe.py C2 >> $OUT/unroll.jsonl 2>&1; done
