#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest_gpu9.log 2>&1
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke9.log 2>&1
timeout 1500 python bench.py > $OUT/bench9.json 2> $OUT/bench9.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_update_fp -s 20 -c 2 \
    -f -o $OUT/prof_update python scripts/profile_run.py C3 30 > $OUT/ncu_upd.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file $OUT/launches_bench_hostloop9.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra --host-loop \
    > $OUT/bench_ncu_hostloop9.log 2>&1
