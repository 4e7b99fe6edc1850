mkdir -p gpurun_out
T=r02h
for k in 0 1 2 3 4 5; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-c5 --degrees 2-4 --option c2_kernel=v6 --option v6_cfg=$k > gpurun_out/${T}_cfg$k.json 2>&1
done
timeout 300 python tools/sanitize_cases.py c2 > gpurun_out/${T}_c2cases.log 2>&1
for k in 1 2 3 4 5; do
  SFK_V6_CFG=$k timeout 300 python -c "
import sys; sys.argv=['x','c2']
from paper_1711_02473_b200 import runtime; runtime.set_option('v6_cfg', $k)
exec(open('tools/sanitize_cases.py').read())
" 2>&1 | grep v6 >> gpurun_out/${T}_c2cases_cfg.log
done
echo fin
