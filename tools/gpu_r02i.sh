python bench.py > gpurun_out/r02i_bench.log 2> gpurun_out/r02i_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r02i_bench.log
