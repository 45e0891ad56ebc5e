#!/bin/bash
# A/B timing of library variants in one GPU session: tools/ab_libs.sh <suffix>...
# (paper_1409_7474_b200/_lib/liblse_b200<suffix>.so; "" = the default build)
for rep in 1 2; do
  for v in "$@"; do
    lib=$PWD/paper_1409_7474_b200/_lib/liblse_b200$v.so
    echo "== lib$v rep $rep"
    LSE_LIB_PATH=$lib python tools/small_probe.py C2 C3 --reps 1 2>&1 | grep "rep 0"
    LSE_LIB_PATH=$lib python tools/c4_probe.py 256 1024 200 2>&1 | tail -1 | sed 's/.*advance/advance/'
    LSE_LIB_PATH=$lib bash tools/quick_bench.sh
  done
done
