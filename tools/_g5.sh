mkdir -p gpurun_out
T=r02f
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "every_kernel_generation" > gpurun_out/${T}_gen.log 2>&1
for k in 0 1; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --degrees 3-8 --option c2_kernel=v6 --option v6_cfg=$k > gpurun_out/${T}_cfg$k.json 2>&1
done
for p in 5 7; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:hex_laplace_action_v6 -s 1 -c 1 -o gpurun_out/${T}_p$p python bench.py --steps 1 --warmup 1 --degrees $p --no-e2e --no-cpu --no-c5 --option c2_kernel=v6 > gpurun_out/${T}_ncu_p$p.log 2>&1
done
echo fin
