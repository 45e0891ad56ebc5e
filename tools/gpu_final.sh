#!/bin/bash
# Round-2 final measurements: full bench, ncu of the fused C5 pass (full set +
# launch list), ncu of the resident kernel (C1) and the small-config launch lists.
mkdir -p gpurun_out
python bench.py > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "bench rc=$?"
bash tools/profile_fused.sh r02y
ncu --set full --clock-control none --import-source on -k regex:k_resident -s 2 -c 1 \
    -o gpurun_out/r02y_resident python tools/small_probe.py C1 --reps 3 > gpurun_out/r02y_ncu_res.log 2>&1
echo "resident full rc=$?"
ncu -i gpurun_out/r02y_resident.ncu-rep --page details > gpurun_out/r02y_resident_details.txt
rm -f gpurun_out/r02y_resident.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02y_small_launches.csv python tools/small_probe.py C1 C2 --reps 2 \
    > gpurun_out/r02y_ncu_small.log 2>&1
echo "small launches rc=$?"
ls -la gpurun_out/r02y_*
