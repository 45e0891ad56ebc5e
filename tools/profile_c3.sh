#!/bin/bash
# ncu --set full of one late-run launch of a C3 kernel (regex $1) -> <tag>_details.txt / _sass.csv
k=$1; tag=$2; skip=${3:-200}
ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/${tag} python tools/c3_phase.py 4096 300 300 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/${tag}.ncu-rep --page details > gpurun_out/${tag}_details.txt
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
