#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest_gpu17.log 2>&1
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke17.log 2>&1
timeout 1500 python bench.py > $OUT/bench17.json 2> $OUT/bench17.err
timeout 300 python scripts/c3_trace.py C3 > $OUT/c3_trace.jsonl 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_symv_bulk -s 3 -c 1 -f -o $OUT/prof_symv_c5_17 python scripts/c5_probe.py 3 > $OUT/ncu_c5_17.log 2>&1
