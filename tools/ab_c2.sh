#!/bin/bash
# A/B: C2 parity tests + bench for hex action kernel variants
TAG=${1:-ab}
mkdir -p gpurun_out
for cfg in "SFK_C2_R=1 SFK_C2_ROLL=1" "SFK_C2_R=1 SFK_C2_ROLL=2" "SFK_C2_R=2"; do
  env $cfg timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c2" >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest $cfg rc=$?" >> gpurun_out/${TAG}_pytest.log
done
SFK_C2_KERNEL=v1 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_v1.json 2>&1
SFK_C2_R=1 SFK_C2_ROLL=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_r1.json 2>&1
SFK_C2_R=1 SFK_C2_ROLL=2 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_r1roll2.json 2>&1
SFK_C2_R=2 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_r2.json 2>&1
