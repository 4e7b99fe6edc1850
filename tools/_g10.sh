mkdir -p gpurun_out
T=r02k
timeout 300 python tools/sanitize_cases.py c2 > gpurun_out/${T}_c2cases.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-c5 --degrees 7 --option c2_kernel=tc8c > gpurun_out/${T}_tc8c.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc8c -s 1 -c 1 -o gpurun_out/${T}_p7 python bench.py --steps 1 --warmup 1 --degrees 7 --no-e2e --no-cpu --no-c5 --option c2_kernel=tc8c > gpurun_out/${T}_ncu_p7.log 2>&1
echo fin
