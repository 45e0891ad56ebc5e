set -x
free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02a_pytest.log
python tools/certify.py --config C5 --out gpurun_out/r02a_certify_c5.json > gpurun_out/r02a_certify_c5.log 2>&1; echo "cert rc=$?"; tail -3 gpurun_out/r02a_certify_c5.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/r02a_bench.log | cut -c1-3000
