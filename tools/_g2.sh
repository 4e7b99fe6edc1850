mkdir -p gpurun_out
T=r02c
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "every_kernel_generation" > gpurun_out/${T}_gen.log 2>&1
timeout 300 python tools/event_overhead.py 1,2,3,4 > gpurun_out/${T}_evoh.jsonl 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --flush dirty > gpurun_out/${T}_dirty.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 > gpurun_out/${T}_clean.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-c5 --degrees 3-8 --option c2_kernel=v6 > gpurun_out/${T}_v6.json 2>&1
echo fin
