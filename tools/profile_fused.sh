#!/bin/bash
# ncu captures of the fused iteration on C5 (dense): one k_update_fused with
# --set full (source/SASS), and the launch list of a short job.
tag=${1:-r02c}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_update_fused -s 30 -c 1 \
    -o gpurun_out/${tag}_fused python bench.py --steps 1 --warmup 1 --iters 20 --no-e2e \
    --no-cpu-baseline --skip-steps 0 --c4-tiles 0 --dropin-steps 0 > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/${tag}_fused.ncu-rep --page raw --csv > gpurun_out/${tag}_fused_raw.csv
ncu -i gpurun_out/${tag}_fused.ncu-rep --page details > gpurun_out/${tag}_fused_details.txt
ncu -i gpurun_out/${tag}_fused.ncu-rep --page source --csv --print-source sass \
    > gpurun_out/${tag}_fused_sass.csv 2>/dev/null
rm -f gpurun_out/${tag}_fused.ncu-rep
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 1 \
    --iters 40 --no-e2e --no-cpu-baseline --skip-steps 0 --c4-tiles 0 --dropin-steps 0 \
    > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launches rc=$?"
ls -la gpurun_out/${tag}_*
