#!/bin/bash
# Full measurement snapshot: tests, smoke, bench (C2 contract), all configs, launch list, p=8 capture
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 1500 python tools/bench_configs.py C1 C3 C4 C5 C2G > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
timeout 600 python tools/bench_programs.py > gpurun_out/${TAG}_lp.jsonl 2> gpurun_out/${TAG}_lp.err
timeout 900 python tools/bench_csr.py > gpurun_out/${TAG}_csr.jsonl 2> gpurun_out/${TAG}_csr.err
bash tools/dist_check.sh
PCMD="python bench.py --steps 1 --warmup 1 --degrees 1-8 --no-e2e --no-cpu"
timeout 600 $PCMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $PCMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
FCMD="python bench.py --steps 1 --warmup 1 --degrees 8 --no-e2e --no-cpu"
timeout 600 $FCMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hex_laplace_action \
    -s 1 -c 1 -o gpurun_out/${TAG}_prof_p8 $FCMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
