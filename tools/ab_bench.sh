cd /root/repo
for rep in 1 2; do for v in base fusexf; do
  echo "== $v c3 rep$rep"; OSAM_LIB=var/$v.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-largest 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['schwarz_steps_per_s'], d['roofline']['k1_ms_per_launch'], d['roofline']['frac'])"
  echo "== $v c4 rep$rep"; OSAM_LIB=var/$v.so timeout 300 python bench.py --workload c4 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e --no-largest 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['schwarz_steps_per_s'], d['roofline']['k1_ms_per_launch'], d['roofline']['frac'])"
done; done
