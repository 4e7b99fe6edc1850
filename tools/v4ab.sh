#!/bin/bash
# A/B of the warp-synchronous C2 kernel (v4) CTA sizes: bash tools/v4ab.sh TAG "libs"
TAG=$1; LIBS=$2
mkdir -p gpurun_out
for lib in $LIBS; do
  if [ "$lib" = "cur" ]; then L=""; else L="$PWD/paper_1711_02473_b200/libsfk_$lib.so"; fi
  SFK_LIBRARY=$L SFK_C2_KERNEL=v4 timeout 300 python tools/bench_configs.py C2 --p 2 3 4 --no-cpu > gpurun_out/${TAG}_v4_$lib.jsonl 2>&1
done
timeout 300 python tools/bench_configs.py C2 --p 2 3 4 --no-cpu > gpurun_out/${TAG}_default.jsonl 2>&1
