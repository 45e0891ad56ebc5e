#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (every kernel family on small inputs, each result checked); logs to gpurun_out/.
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py > "$out/plain.log" 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 200 python tools/sanitize_cases.py \
      > "$out/$tool.log" 2>&1
  echo "$tool rc=$?"; tail -4 "$out/$tool.log"
done
