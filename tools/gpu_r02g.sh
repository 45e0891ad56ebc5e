python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider > gpurun_out/r02g_fused.log 2>&1; echo "fused rc=$?"; tail -3 gpurun_out/r02g_fused.log
bash tools/ab_c5.sh "" "_f4"
