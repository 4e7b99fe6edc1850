mkdir -p gpurun_out
T=r02g
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-c5 --degrees 3-6 --option c2_kernel=v6 --option v6_cfg=4 > gpurun_out/${T}_zr.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --degrees 3-8 --option c2_kernel=v6 > gpurun_out/${T}_v6.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --degrees 3-8 > gpurun_out/${T}_auto.json 2>&1
echo fin
