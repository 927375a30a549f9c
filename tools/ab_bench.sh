#!/bin/bash
# A/B timing on one box: every ab/*.so (OSAM_LIB) x every env setting in VARENV, c3 and c4, REPS rounds
# (bench.py, no ncu).  Usage: VARENV="X=0 OSAM_SERIAL_K1=1" REPS=2 bash tools/ab_bench.sh
cd "$(dirname "$0")/.."
VARENV=${VARENV:-"X=0"}
REPS=${REPS:-1}
LIBS=$(ls ab/*.so 2>/dev/null || echo paper_2511_20687_b200/libosam.so)
for rep in $(seq $REPS); do for v in $LIBS; do for e in $VARENV; do
  for w in ${WORKLOADS:-c3 c4}; do
    r=$(env $e OSAM_LIB=$v timeout 300 python bench.py --workload $w --steps 80 --warmup 5 --no-cpu-baseline --no-e2e --no-largest 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['schwarz_steps_per_s'],1), 'iters', d['schwarz_iters_per_step'], 'k1_busy/step', round(r.get('k1_busy_ms_per_step',0),4), 'k1/launch', round(r['k1_ms_per_launch'],4), 'serial', round(r.get('serial_profile',{}).get('k1_ms_per_launch',0),4))")
    echo "$v $e $w rep$rep $r"
  done
done; done; done
