#!/bin/bash
# A/B of alternative builds of libsfk (same ABI): bash tools/ab_libs.sh TAG "cur ab ..." [bench args]
TAG=$1; LIBS=$2; shift 2
mkdir -p gpurun_out
for lib in $LIBS; do
  if [ "$lib" = "cur" ]; then L=""; else L="$PWD/paper_1711_02473_b200/libsfk_$lib.so"; fi
  SFK_LIBRARY=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu "$@" > gpurun_out/${TAG}_${lib}.json 2>&1
done
