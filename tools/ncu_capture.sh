#!/bin/bash
# ncu evidence for profiles/: (a) every K1 kernel of one c3 controller step (3 sweeps x (Omega1 tiled,
# Omega2 tiled, Omega2 x-face)) with --set full; (b) one c5 DMMA GEMM with --set full.
# Each command first runs without ncu (exit 0 required), as the profiling recipe asks.
TAG=${1:-r}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export OSAM_NOGRAPH=1  # ncu cannot profile kernel nodes of graphs with conditional nodes
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-largest"
timeout 600 $B > gpurun_out/cap_plain_$TAG.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:fom_ -s 30 -c 9 -o gpurun_out/k1step_$TAG $B > gpurun_out/cap_ncu_$TAG.log 2>&1
C="python tools/bench_configs.py c5"
STEPS=3 timeout 600 $C > gpurun_out/cap_plain_c5_$TAG.log 2>&1 && \
  STEPS=3 timeout 900 ncu --set full --clock-control none -k regex:dmma_gemm -s 40 -c 2 -o gpurun_out/dmma_$TAG $C > gpurun_out/cap_ncu_c5_$TAG.log 2>&1
echo done
