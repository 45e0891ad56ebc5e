#!/bin/bash
# ncu --set full of one launch of a kernel (regex $1, skipping $2 launches) in a
# short C5 job; exported on the box: <tag>_raw.csv, _details.txt, _sass.csv
k=$1; skip=${2:-30}; tag=${3:-prof}; iters=${4:-60}
ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/${tag} python bench.py --steps 1 --warmup 1 --iters $iters --no-e2e \
    --no-cpu-baseline --skip-steps 0 --c4-tiles 0 --dropin-steps 0 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i gpurun_out/${tag}.ncu-rep --page details > gpurun_out/${tag}_details.txt
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
