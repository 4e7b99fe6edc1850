#!/bin/bash
# Repeated A/B of library builds on bench_configs: bash tools/ab_cfg_rep.sh TAG "cur lib2 ..." REPS CFG [args]
TAG=$1; LIBS=$2; REPS=$3; CFG=$4; shift 4
mkdir -p gpurun_out
for r in $(seq 1 $REPS); do
  for lib in $LIBS; do
    if [ "$lib" = "cur" ]; then L=""; else L="$PWD/paper_1711_02473_b200/libsfk_$lib.so"; fi
    SFK_LIBRARY=$L timeout 600 python tools/bench_configs.py $CFG --no-cpu "$@" >> gpurun_out/${TAG}_${lib}.jsonl 2>>gpurun_out/${TAG}.err
  done
done
