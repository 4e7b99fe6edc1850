#!/bin/bash
# Repeated interleaved A/B of library builds: bash tools/ab_rep.sh TAG "cur lib2 ..." REPS [bench args]
TAG=$1; LIBS=$2; REPS=$3; shift 3
mkdir -p gpurun_out
for r in $(seq 1 $REPS); do
  for lib in $LIBS; do
    if [ "$lib" = "cur" ]; then L=""; else L="$PWD/paper_1711_02473_b200/libsfk_$lib.so"; fi
    SFK_LIBRARY=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu "$@" >> gpurun_out/${TAG}_${lib}.jsonl 2>>gpurun_out/${TAG}.err
  done
done
