#!/bin/bash
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for V in sr16 sr16s4; do
  for W in C3 C5; do
    IPM_LIB=$PWD/paper_2405_03584_b200/libipm_$V.so timeout 600 python scripts/symv_order_probe.py $W | sed "s/^{/{\"variant\": \"$V\", /" >> $OUT/sr.jsonl 2>&1
  done
done
for W in C3 C5; do timeout 600 python scripts/symv_order_probe.py $W | sed "s/^{/{\"variant\": \"sr32\", /" >> $OUT/sr.jsonl 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_c4.py -q -x > $OUT/pytest16.log 2>&1
timeout 1000 python scripts/c4_sequence.py 8 > $OUT/c4p_warm8.jsonl 2>&1
timeout 2100 python scripts/c4_sequence.py 30 --cold > $OUT/c4p_cold30.jsonl 2>&1
