#!/bin/bash
# One parameterised GPU-side profiling runner (run under gpurun from the repo root).
#   scripts/gpu_profile.sh symv <workload> <tag>   ncu --set full of the PCG-mode SYMV (1 launch)
#   scripts/gpu_profile.sh spmv <workload> <tag>   ncu --set full of the PCG-mode SpMV / SpMV^T
#   scripts/gpu_profile.sh launches <workload> <tag>   launch list of the bench command (host-loop PCG)
set -x
mode=$1; wl=${2:-C5}; tag=${3:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
case $mode in
symv)
  # skip the residual-mode (<0>) launch of the first residuals; capture the first PCG-mode launch
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_symv_bulk -s 1 -c 1 \
      -o gpurun_out/${tag}_${wl}_symv -f python scripts/profile_run.py $wl 4 > gpurun_out/${tag}_${wl}_symv.log 2>&1
  ncu -i gpurun_out/${tag}_${wl}_symv.ncu-rep --page raw --csv > gpurun_out/${tag}_${wl}_symv_raw.csv 2>&1
  ;;
spmv)
  # the PCG-mode SpMV and SpMV^T of the host-loop PCG (2 launches each)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 4 \
      -o gpurun_out/${tag}_${wl}_spmv -f python scripts/profile_run.py $wl 4 > gpurun_out/${tag}_${wl}_spmv.log 2>&1
  ncu -i gpurun_out/${tag}_${wl}_spmv.ncu-rep --page raw --csv > gpurun_out/${tag}_${wl}_spmv_raw.csv 2>&1
  ;;
launches)
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -s ${SKIP:-400} -c ${COUNT:-800} --csv --log-file gpurun_out/${tag}_${wl}_launches.csv \
      python bench.py --workload $wl --host-loop --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
      > gpurun_out/${tag}_${wl}_launches.log 2>&1
  ;;
esac
