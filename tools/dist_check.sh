#!/bin/bash
# torchrun launch paths of bench.py (1 GPU box: nproc 1) + the reference arm
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/dist_bench.json 2> gpurun_out/dist_bench.err
echo "torchrun bench rc=$?" >> gpurun_out/dist_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_bench.json 2> gpurun_out/ref_bench.err
echo "reference rc=$?" >> gpurun_out/ref_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/ref_dist.json 2> gpurun_out/ref_dist.err
echo "reference torchrun rc=$?" >> gpurun_out/ref_dist.err
timeout 600 python bench.py --scaling strong --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/strong_bench.json 2> gpurun_out/strong_bench.err
echo "strong rc=$?" >> gpurun_out/strong_bench.err
