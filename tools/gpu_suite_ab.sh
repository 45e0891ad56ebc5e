#!/bin/bash
# whole GPU suite + C5 A/B of the given builds + launch list
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/suite.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/suite.log
bash tools/ab_c5.sh "$@"
