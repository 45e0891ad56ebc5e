ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_spec_fix -s 8 -c 1 \
    -o gpurun_out/fix3 python bench.py --steps 1 --warmup 1 --iters 30 --no-e2e \
    --no-cpu-baseline --skip-steps 0 --c4-tiles 0 --dropin-steps 0 > gpurun_out/fix3_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/fix3.ncu-rep --page details > gpurun_out/fix3_details.txt
ncu -i gpurun_out/fix3.ncu-rep --page source --csv --print-source sass > gpurun_out/fix3_sass.csv 2>/dev/null
rm -f gpurun_out/fix3.ncu-rep
