python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider > gpurun_out/r02e_fused.log 2>&1; echo "fused rc=$?"; tail -3 gpurun_out/r02e_fused.log
bash tools/ab_c5.sh "" "_np" "_pf" "|LSE_FUSED=0"
