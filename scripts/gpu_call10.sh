#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest_gpu10.log 2>&1
timeout 600 ./scripts/micro/stream_bw 100000 > $OUT/stream_bw_1e5.jsonl 2>&1
timeout 900 python scripts/c5_probe.py 3 > $OUT/c5_probe.jsonl 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_symv_bulk -s 3 -c 1 -f -o $OUT/prof_symv_c5 python scripts/c5_probe.py 3 > $OUT/ncu_c5.log 2>&1
timeout 2700 python scripts/c4_sequence.py 30 > $OUT/c4_warm.jsonl 2>&1
