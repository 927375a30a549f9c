cd /root/repo
for rep in 1; do for v in ab/*.so; do for m in svk neohookean; do
  r=$(OSAM_LIB=$v timeout 300 python bench.py --material $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-largest 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['schwarz_steps_per_s'],1), round(r['k1_ms_per_launch'],4), round(r['frac'],4))")
  echo "$v $m rep$rep $r"
done; done; done
