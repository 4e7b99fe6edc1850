#!/bin/bash
# ncu --set full of the C2 kernel at given degrees: bash tools/prof.sh TAG "8 4" [ENV...]
TAG=$1; DEGS=$2; shift 2
mkdir -p gpurun_out
for p in $DEGS; do
  CMD="python bench.py --steps 1 --warmup 1 --degrees $p --no-e2e --no-cpu"
  env "$@" timeout 600 $CMD > gpurun_out/${TAG}_plain_p$p.log 2>&1 && \
  env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:hex_laplace_action \
     -s 1 -c 1 -o gpurun_out/${TAG}_p$p $CMD > gpurun_out/${TAG}_ncu_p$p.log 2>&1
done
