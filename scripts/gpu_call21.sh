#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
IPM_DEBUG=1 timeout 4400 python scripts/c5_solve.py > $OUT/c5_solve.jsonl 2> $OUT/c5_solve.err
echo "exit $?" >> $OUT/c5_solve.err
