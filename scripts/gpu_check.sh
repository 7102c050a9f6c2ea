#!/bin/bash
# One gpurun call: build, GPU test suite, smoke, default bench, launch list + full ncu capture
# of the dominant kernel.  Everything lands in gpurun_out/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > $OUT/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.log
  timeout 300 python __graft_entry__.py --smoke > $OUT/smoke.log 2>&1
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
  timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
fi
if [ "${SKIP_NCU:-0}" != 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${NCU_SKIP:-3000} -c 400 --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra \
    > $OUT/bench_under_ncu.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_symv_bulk -s 20 -c 2 \
    -f -o $OUT/prof_symv python scripts/profile_run.py C3 30 > $OUT/ncu_full.log 2>&1
fi
