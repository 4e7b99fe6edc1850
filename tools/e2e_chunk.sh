#!/bin/bash
# e2e staging chunk size A/B: bash tools/e2e_chunk.sh TAG "16 32 64 128" REPS
TAG=$1; SIZES=$2; REPS=${3:-2}
mkdir -p gpurun_out
for r in $(seq 1 $REPS); do
  for mb in $SIZES; do
    SFK_HOST_CHUNK_MB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu >> gpurun_out/${TAG}_${mb}.jsonl 2>>gpurun_out/${TAG}.err
  done
done
