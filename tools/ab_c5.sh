#!/bin/bash
# C5 headline A/B of library builds (and LSE_* settings) on one box:
#   tools/ab_c5.sh "<suffix>|<ENV=VAL ...>" ...   ("" = default build)
for rep in 1 2; do
  for spec in "$@"; do
    v=${spec%%|*}; e=""; [[ "$spec" == *"|"* ]] && e=${spec#*|}
    echo -n "lib$v [$e] rep $rep: "
    env $e LSE_LIB_PATH=$PWD/paper_1409_7474_b200/_lib/liblse_b200$v.so bash tools/quick_bench.sh
  done
done
