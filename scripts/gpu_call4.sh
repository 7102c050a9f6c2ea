#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest_gpu4.log 2>&1
for F in 0 1; do
  IPM_FUSED_P=$F PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/fused.jsonl 2>&1
  IPM_FUSED_P=$F timeout 300 python scripts/pcg_iter_probe.py C2 >> $OUT/fused.jsonl 2>&1
  IPM_FUSED_P=$F timeout 300 python scripts/pcg_iter_probe.py C1 >> $OUT/fused.jsonl 2>&1
done
timeout 1500 python bench.py > $OUT/bench4.json 2> $OUT/bench4.err
