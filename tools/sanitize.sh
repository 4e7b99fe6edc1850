#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over small
# launches of every kernel family: bash tools/sanitize.sh TAG [FAMILIES...]
TAG=${1:-r02}; shift
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --version > gpurun_out/${TAG}_sanitizer_version.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py "$@" > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "exit=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
done
