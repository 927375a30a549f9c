#!/bin/bash
# ncu launch list + full capture of the K1 tiled kernel (one launch of each subdomain) for bench.py c3
TAG=${1:-r}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export OSAM_NOGRAPH=1  # ncu cannot profile kernel nodes of graphs with conditional nodes
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-largest"
timeout 300 $B > gpurun_out/plain_$TAG.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fom_tiled -s 6 -c 2 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu2_$TAG.log 2>&1
echo done
