# same-box A/B of the generation loop: ab_old/ (a previous commit's package,
# built) vs the working tree, alternating the order (power-capped box), for
# the configs in ABCFGS
for rep in 1 2 3 4; do
  if [ $((rep % 2)) = 1 ]; then SIDES='old new'; else SIDES='new old'; fi
  for side in $SIDES; do
    for c in ${ABCFGS:-c2 c3}; do
      if [ $side = old ]; then B=ab_old/bench.py; else B=bench.py; fi
      timeout 600 python $B --config $c --steps ${ABSTEPS:-30} --warmup 5 --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 > gpurun_out/ab_${side}_$c.json
      python -c "
import json; d=json.load(open('gpurun_out/ab_${side}_$c.json'))
print('$rep $side $c', round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline'].get('kernel_share_of_step',0),4), d['clocks']['sm_mhz'])"
    done
  done
done
