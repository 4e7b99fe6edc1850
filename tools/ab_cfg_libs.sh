#!/bin/bash
# A/B of alternative builds on tools/bench_configs.py: bash tools/ab_cfg_libs.sh TAG "cur ab" CONFIGS...
TAG=$1; LIBS=$2; shift 2
mkdir -p gpurun_out
for lib in $LIBS; do
  if [ "$lib" = "cur" ]; then L=""; else L="$PWD/paper_1711_02473_b200/libsfk_$lib.so"; fi
  SFK_LIBRARY=$L timeout 900 python tools/bench_configs.py "$@" --no-cpu > gpurun_out/${TAG}_${lib}.jsonl 2>&1
done
