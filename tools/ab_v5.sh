set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_kernel_generation or c2_" > gpurun_out/r01bu_pytest.log 2>&1; echo rc=$? >> gpurun_out/r01bu_pytest.log
for r in 1 2; do
for cfg in "X=0" "SFK_C2_KERNEL=v5 SFK_C2_G=1" "SFK_C2_KERNEL=v5 SFK_C2_G=2" "SFK_C2_KERNEL=v5 SFK_C2_G=3"; do
  name=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --degrees 4-6,8 >> gpurun_out/r01bu_$name.jsonl 2>>gpurun_out/r01bu.err
done; done
