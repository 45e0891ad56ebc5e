#!/bin/bash
# Round profile capture on the GPU box (run from the repo root):
#   1. the bench line itself (no profiler)
#   2. the launch list of the same command (ncu, per-launch duration, cold, serialised)
#   3. ncu --set full of one steady-state k_update and k_partition (C5, dense)
set -e
tag=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --c4-tiles 0 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_bench.log 2>&1
for k in k_update k_partition; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 25 -c 1 \
      -o gpurun_out/${tag}_$k python bench.py --steps 1 --warmup 1 --iters 20 --no-e2e \
      --no-cpu-baseline --skip-steps 0 --c4-tiles 0 > /dev/null 2>&1
done
# export on the box (reports with source are too big to travel back whole)
for k in k_update k_partition; do
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_${k}_raw.csv
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page details > gpurun_out/${tag}_${k}_details.txt
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page source --csv --print-source sass \
      > gpurun_out/${tag}_${k}_sass.csv 2>/dev/null
  rm -f gpurun_out/${tag}_$k.ncu-rep
done
ls -la gpurun_out/${tag}_*
