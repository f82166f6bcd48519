# GSM A/B: gsm_alt/base.so vs gsm_alt/new.so (alternating, 2 reps)
set -x
O=gpurun_out/${AB_OUT:-r02/ab_gsm2}; mkdir -p $O
for rep in 1 2; do
for lib in gsm_alt/base.so gsm_alt/new.so; do
  for c in ${AB_CFGS:-c3 c5 c4 c2}; do
    st=30; [ $c = c2 ] && st=300
    r=$(GSGP_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))")
    echo "$rep $lib $c $r" | tee -a $O/ab.log
  done
done
done
