#!/bin/bash
# ncu --set full of several kernels, summarised ON THE BOX (the .ncu-rep files
# are too large to bring back together): bash tools/prof_batch.sh TAG
TAG=$1
mkdir -p gpurun_out/${TAG}_md
bash tools/prof.sh $TAG "1 2 3 4 5 6 7"
bash tools/prof_cfg.sh $TAG C3 8 hex_colloc
bash tools/prof_cfg.sh $TAG C3 15 hex_colloc
bash tools/prof_cfg.sh $TAG C5 3 hex_laplace_matrix
bash tools/prof_cfg.sh $TAG C5 4 hex_laplace_matrix
bash tools/prof_cfg.sh $TAG C4 6 hex_neohookean
for r in gpurun_out/${TAG}_*.ncu-rep; do
  k=$(basename $r .ncu-rep)
  python tools/ncu_summary.py $r "$k" > /dev/null 2>&1
  cp profiles/$k.md gpurun_out/${TAG}_md/ 2>/dev/null
  rm -f $r
done
cp profiles/ncu_traffic.json gpurun_out/${TAG}_md/
