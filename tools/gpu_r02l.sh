timeout 600 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/r02l_bands.log 2>&1; echo "bands rc=$?"; tail -3 gpurun_out/r02l_bands.log
timeout 300 python tools/c3_phase.py 4096 1000 50 > gpurun_out/r02l_c3_phase.log 2>&1; echo "phase rc=$?"; cat gpurun_out/r02l_c3_phase.log | tail -6
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 60 --csv --log-file gpurun_out/r02l_c3_late.csv python tools/c3_phase.py 4096 1000 1000 > /dev/null 2>&1; echo "ncu rc=$?"
