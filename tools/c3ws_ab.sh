#!/bin/bash
# C3 warp-synchronous mode A/B (n <= 5): bash tools/c3ws_ab.sh TAG
TAG=$1
mkdir -p gpurun_out
SFK_COLLOC_WARPS=8 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_assembly.py -q -m gpu -k "c3 or collocated" > gpurun_out/${TAG}_pytest_w8.log 2>&1
for w in 0 8; do
  SFK_COLLOC_WARPS=$w timeout 600 python tools/bench_configs.py C3 C3G --p 4 --no-cpu > gpurun_out/${TAG}_w$w.jsonl 2>&1
done
