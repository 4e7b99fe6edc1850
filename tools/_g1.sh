set -x
mkdir -p gpurun_out
bash tools/gpu_check.sh r02b
timeout 300 python tools/event_overhead.py 1,2,3,4 > gpurun_out/r02b_evoh.jsonl 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --flush dirty > gpurun_out/r02b_dirty.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --flush clean > gpurun_out/r02b_clean.json 2>&1
echo fin
