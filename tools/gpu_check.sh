#!/bin/bash
# gpurun session: GPU tests (no -x: every failure), smoke, default bench.
# usage (repo root on the GPU box): bash tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-r02}
K=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc >> gpurun_out/${TAG}_smi.txt
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$K" --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
echo done
