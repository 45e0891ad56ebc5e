#!/bin/bash
# A/B of library variants on sizes that use the per-pixel kernels by default
for rep in 1 2; do for v in "$@"; do echo "== lib$v"; LSE_LIB_PATH=$PWD/paper_1409_7474_b200/_lib/liblse_b200$v.so python tools/small_probe.py C1 X384 X512 --reps 2 2>&1 | grep "rep 1"; done; done
