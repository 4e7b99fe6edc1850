#!/bin/bash
TAG=${1:-ab}
mkdir -p gpurun_out
for cfg in "SFK_C2_KERNEL=v2 SFK_C2_CPB=0" "SFK_C2_KERNEL=v2 SFK_C2_CPB=4" "SFK_C2_KERNEL=v2 SFK_C2_CPB=12" "SFK_C2_KERNEL=v2 SFK_C2_CPB=8" "SFK_C2_KERNEL=v2 SFK_C2_CPB=5"; do
  name=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --degrees 5,6,8 > gpurun_out/${TAG}_$name.json 2>&1
done
