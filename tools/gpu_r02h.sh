python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/r02h_pytest.log
bash tools/quick_bench.sh
bash tools/profile_fused.sh r02h
