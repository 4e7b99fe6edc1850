#!/bin/bash
# A/B: C2 parity tests + bench for hex action kernel variants
TAG=${1:-ab}
mkdir -p gpurun_out
for cfg in "SFK_C2_KERNEL=tc"; do
  env $cfg timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c2" >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest $cfg rc=$?" >> gpurun_out/${TAG}_pytest.log
done
SFK_C2_KERNEL=tc timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --degrees 7 > gpurun_out/${TAG}_tc.json 2>&1
