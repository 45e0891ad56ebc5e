python -m pytest tests/test_gpu_batch.py tests/test_gpu_fused.py -x -q -p no:cacheprovider > gpurun_out/c4ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c4ab_tests.log
for rep in 1 2; do
python tools/c4_probe.py 256 1024 300 2>&1 | tail -1
LSE_FUSED=0 python tools/c4_probe.py 256 1024 300 2>&1 | tail -1
done
