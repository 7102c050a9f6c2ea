#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for O in 0 1; do IPM_SYM_ORDER=$O timeout 300 python scripts/symv_order_probe.py C3 >> $OUT/order.jsonl 2>&1; done
for O in 0 1; do IPM_SYM_ORDER=$O timeout 300 python scripts/symv_order_probe.py C2 >> $OUT/order.jsonl 2>&1; done
for O in 0 1; do IPM_SYM_ORDER=$O timeout 600 python scripts/symv_order_probe.py C5 >> $OUT/order.jsonl 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "symmetric" > $OUT/pytest15.log 2>&1
