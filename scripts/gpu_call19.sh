#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python paper_2405_03584_b200/build.py --timeline >> $OUT/build.log 2>&1
timeout 300 python scripts/timeline_probe.py C3 > $OUT/timeline_c3_19.log 2>&1
PROBE_QP=0 timeout 300 python scripts/pcg_iter_probe.py C3 >> $OUT/probe19.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -q --durations=5 > $OUT/pytest_gpu19.log 2>&1
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke19.log 2>&1
timeout 1500 python bench.py > $OUT/bench19.json 2> $OUT/bench19.err
