#!/bin/bash
# ncu --set full of the Schwarz transfer (separate launches, OSAM_XFER_INGRID=0) and of the tiled K1 with the
# in-grid transfer, c3 host-driven sweeps (ncu cannot profile graphs with conditional nodes)
TAG=${1:-r}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export OSAM_NOGRAPH=1
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-largest"
OSAM_XFER_INGRID=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:transfer_kernel -s 8 -c 2 -o gpurun_out/xfer_$TAG $B > gpurun_out/ncu_xfer_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fom_tiled -s 8 -c 2 -o gpurun_out/k1in_$TAG $B > gpurun_out/ncu_k1in_$TAG.log 2>&1
echo done
