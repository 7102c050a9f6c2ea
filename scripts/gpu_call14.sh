#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --durations=15 > $OUT/pytest_gpu14.log 2>&1
timeout 300 python __graft_entry__.py --smoke > $OUT/smoke14.log 2>&1
timeout 1500 python bench.py > $OUT/bench14.json 2> $OUT/bench14.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench14_ref.json 2> $OUT/bench14_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling graph --csv \
    --log-file $OUT/launches14_graphs.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra \
    > $OUT/bench14_ncu_graphs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file $OUT/launches14_hostloop.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra --host-loop \
    > $OUT/bench14_ncu_hostloop.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_symv_bulk -s 20 -c 2 \
    -f -o $OUT/prof_symv14 python scripts/profile_run.py C3 30 > $OUT/ncu_symv14.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_pcg_update_fp -s 20 -c 2 \
    -f -o $OUT/prof_update14 python scripts/profile_run.py C3 30 > $OUT/ncu_upd14.log 2>&1
timeout 2400 python scripts/c4_sequence.py 30 --cold > $OUT/c4_cold.jsonl 2>&1
