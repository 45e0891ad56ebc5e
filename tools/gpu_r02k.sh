# round-2 re-entry check: GPU suite + full bench on the committed HEAD
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02k_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02k_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02k_bench.log 2> gpurun_out/r02k_bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r02k_bench.log
