#!/bin/bash
# Repeated A/B of environment settings: bash tools/ab_env.sh TAG REPS DEGREES "ENV1" "ENV2" ...
TAG=$1; REPS=$2; DEG=$3; shift 3
mkdir -p gpurun_out
for r in $(seq 1 $REPS); do
  for cfg in "$@"; do
    name=$(echo "$cfg" | tr ' =' '__')
    env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --degrees $DEG >> gpurun_out/${TAG}_${name}.jsonl 2>>gpurun_out/${TAG}.err
  done
done
