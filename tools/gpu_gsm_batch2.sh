# GSM claim batch A/B (GSGP_GSM_BATCH forced) with the in-tree library
set -x
O=gpurun_out/r02/batch; mkdir -p $O
for rep in 1 2; do
for b in default 8 16 32; do
  for c in c4 c3 c5 c2; do
    st=30; [ $c = c2 ] && st=300
    if [ $b = default ]; then unset GSGP_GSM_BATCH; else export GSGP_GSM_BATCH=$b; fi
    r=$(timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
    echo "$rep batch=$b $c $r" | tee -a $O/ab.log
  done
done
done
