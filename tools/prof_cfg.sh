#!/bin/bash
# ncu --set full of one config/degree kernel: bash tools/prof_cfg.sh TAG CFG P REGEX
TAG=$1; CFG=$2; P=$3; RX=$4
mkdir -p gpurun_out
CMD="python tools/bench_configs.py $CFG --p $P --reps 1 --no-cpu"
timeout 600 $CMD > gpurun_out/${TAG}_plain_${CFG}_p$P.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s 1 -c 1 \
   -o gpurun_out/${TAG}_${CFG}_p$P $CMD > gpurun_out/${TAG}_ncu_${CFG}_p$P.log 2>&1
