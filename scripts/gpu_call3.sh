#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sqp.py tests/test_gpu_compact.py -q > $OUT/pytest_sqp.log 2>&1
timeout 600 python scripts/symv_balance.py > $OUT/symv_balance.jsonl 2>&1
for G in 4 8 16 32; do IPM_UPD_G=$G timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/upd_g.jsonl 2>&1; done
timeout 300 python scripts/pcg_iter_probe.py C2 >> $OUT/l2_c2.jsonl 2>&1
IPM_SYM_KEEP_MB=110 timeout 300 python scripts/pcg_iter_probe.py C2 >> $OUT/l2_c2.jsonl 2>&1
PERSIST_MB=100 IPM_SYM_KEEP_MB=110 timeout 300 python scripts/pcg_iter_probe.py C2 >> $OUT/l2_c2.jsonl 2>&1
PERSIST_MB=100 IPM_SYM_KEEP_MB=80 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/l2_c2.jsonl 2>&1
