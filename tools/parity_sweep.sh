#!/bin/bash
# Small-batch parity sweep of every family and every kernel mode switch
TAG=$1
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/${TAG}_sweep.log; env "$@" timeout 600 python tools/parity_sweep.py >> gpurun_out/${TAG}_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_sweep.log; }
run SFK_NONE=1
for g in v1 v2 v3 v4 v5 tc cell cellv; do run SFK_C2_KERNEL=$g; done
for g in 1 2 3; do run SFK_C2_KERNEL=v5 SFK_C2_G=$g; done
run SFK_V5_CPB6=8
run SFK_CELL_TH=128
run SFK_HOST_CHUNK_MB=16
run SFK_COLLOC_WARPS=8
run SFK_C3_TC=1
run SFK_NEO_WARPS=0
run SFK_C5_P1=phase SFK_C5_P3=phase SFK_C5_P4=phase
run SFK_CSR_DMMA=1
run SFK_LP_WARP=0 SFK_LP_FUSE=0
run SFK_C2G_KERNEL=v3
run SFK_C2G_KERNEL=v2
