#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_sqp.py -x -q -k "test_sqp_matches_oracle and 0-1" > $OUT/sanitizer_sqp.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest_gpu2.log 2>&1
timeout 600 python scripts/l2_keep_sweep.py C3 > $OUT/l2_keep.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling graph --csv \
    --log-file $OUT/launches_bench_graphs.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra \
    > $OUT/bench_ncu_graphs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file $OUT/launches_bench_hostloop.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra --host-loop \
    > $OUT/bench_ncu_hostloop.log 2>&1
