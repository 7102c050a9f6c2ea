#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling graph --csv \
    --log-file $OUT/launches20_graphs.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra \
    > $OUT/bench20_ncu_graphs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file $OUT/launches20_hostloop.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra --host-loop \
    > $OUT/bench20_ncu_hostloop.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_symv_bulk -s 20 -c 2 \
    -f -o $OUT/prof_symv20 python scripts/profile_run.py C3 30 > $OUT/ncu_symv20.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_pcg_update_fp -s 20 -c 2 \
    -f -o $OUT/prof_update20 python scripts/profile_run.py C3 30 > $OUT/ncu_upd20.log 2>&1
