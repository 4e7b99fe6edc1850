mkdir -p gpurun_out
T=r02j
timeout 300 python tools/sanitize_cases.py c2 > gpurun_out/${T}_c2cases.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-c5 --degrees 1 --option c2_kernel=p1c > gpurun_out/${T}_p1c.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --degrees 1 > gpurun_out/${T}_p1.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hex_laplace_action -s 1 -c 1 -o gpurun_out/${T}_p1c python bench.py --steps 1 --warmup 1 --degrees 1 --no-e2e --no-cpu --no-c5 --option c2_kernel=p1c > gpurun_out/${T}_ncu_p1c.log 2>&1
echo fin
