#!/bin/bash
# time variant builds ab/*.so with bench.py (no ncu) under the env settings in VARENV
VARENV=${VARENV:-"X=0"}
cd "$(dirname "$0")/.."
for v in ab/*.so; do
  for e in $VARENV; do
    echo "== $v $e"; env $e OSAM_LIB=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-largest 2>&1 | tail -1
  done
done > gpurun_out/var.log 2>&1
