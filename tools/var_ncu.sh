#!/bin/bash
# dram traffic of one K1 tiled launch (Omega1, sweep >= 2) for each variant in ab/
cd "$(dirname "$0")/.."
for v in ab/*.so; do
  n=$(basename $v .so)
  OSAM_LIB=$v timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-largest > gpurun_out/vplain_$n.log 2>&1 && \
  OSAM_LIB=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__average_warp_latency_per_inst_issued.ratio --clock-control none -k regex:fom_tiled -s 8 -c 1 --csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-largest > gpurun_out/vncu_$n.csv 2>&1
done
