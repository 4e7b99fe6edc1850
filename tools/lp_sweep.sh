#!/bin/bash
# Sweep the LoopProgram generator's launch-shape knobs: bash tools/lp_sweep.sh TAG
# (SFK_LP_SMEM_KB: smem budget per CTA; SFK_LP_MAX_THREADS: CTA size cap;
#  SFK_LP_MINB: __launch_bounds__ min blocks)
TAG=$1
timeout 300 python tools/bench_programs.py --reps 5 > gpurun_out/${TAG}_auto.jsonl 2>/dev/null
for t in 128 256 512; do
  for mb in 1 2 4; do
    SFK_LP_MAX_THREADS=$t SFK_LP_MINB=$mb timeout 300 python tools/bench_programs.py --reps 5 \
      > gpurun_out/${TAG}_t${t}_mb${mb}.jsonl 2>/dev/null
  done
done
