#!/bin/bash
# one GPU round: tests, bench, ncu launch list, ncu full capture of the FOM kernels
set -x
TAG=${1:-r}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-largest"
nvidia-smi > gpurun_out/smi_$TAG.txt 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 900 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1
# ncu cannot profile kernel nodes of graphs with conditional nodes: host-driven sweeps for ncu
export OSAM_NOGRAPH=1
timeout 300 $B > gpurun_out/plain_$TAG.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu1_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fom_tiled -s 6 -c 6 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu2_$TAG.log 2>&1
echo done
