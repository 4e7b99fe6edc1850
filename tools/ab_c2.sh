#!/bin/bash
TAG=${1:-ab}
mkdir -p gpurun_out
for cfg in "SFK_C2_KERNEL=v2 SFK_C2_CPB9=2" "SFK_C2_KERNEL=v2 SFK_C2_CPB9=4" "SFK_C2_KERNEL=v3 SFK_C2_V3MINB1=1"; do
  name=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c2 and 8" >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest $cfg rc=$?" >> gpurun_out/${TAG}_pytest.log
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --degrees 8 > gpurun_out/${TAG}_$name.json 2>&1
done
