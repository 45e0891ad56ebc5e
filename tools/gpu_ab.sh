#!/bin/bash
# fused tests with the default build, then C5 A/B of the given builds
python -m pytest tests/test_gpu_fused.py -x -q -p no:cacheprovider > gpurun_out/ab_fused.log 2>&1; echo "fused rc=$?"; tail -2 gpurun_out/ab_fused.log
bash tools/ab_c5.sh "$@"
