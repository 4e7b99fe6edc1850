mkdir -p gpurun_out
T=r02i
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 > gpurun_out/${T}_auto.json 2>&1
for p in 1 2 3 4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:hex_laplace_action -s 1 -c 1 -o gpurun_out/${T}_p$p python bench.py --steps 1 --warmup 1 --degrees $p --no-e2e --no-cpu --no-c5 > gpurun_out/${T}_ncu_p$p.log 2>&1
done
echo fin
