#!/bin/bash
# C4 warp-synchronous mode A/B: bash tools/c4ws_ab.sh TAG
TAG=$1
mkdir -p gpurun_out
for w in 8 4; do
  SFK_NEO_WARPS=$w timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_assembly.py -q -m gpu -k "c4 or neohookean" > gpurun_out/${TAG}_pytest_w$w.log 2>&1
done
for w in 0 4 8; do
  SFK_NEO_WARPS=$w timeout 600 python tools/bench_configs.py C4 C4G --no-cpu > gpurun_out/${TAG}_w$w.jsonl 2>&1
done
