#!/bin/bash
# gpu tests + per-config measurements: bash tools/gpu_tests.sh TAG [configs...] [--p ...]
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
shift
timeout 1500 python tools/bench_configs.py "$@" > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
echo "configs rc=$?" >> gpurun_out/${TAG}_configs.err
