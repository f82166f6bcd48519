# C1 (launch/latency-bound) A/B of ab_old vs the working tree: loop rate, e2e and its init phases
for rep in 1 2; do
  for side in old new; do
    if [ $side = old ]; then B=ab_old/bench.py; else B=bench.py; fi
    timeout 600 python $B --config c1 --steps 200 --warmup 5 --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 > gpurun_out/abc1.json
    python -c "
import json; d=json.load(open('gpurun_out/abc1.json')); e=d['e2e']
print('$rep $side', round(d['value'],1), 'step_us', round(d['ms_per_step']*1000,2), 'e2e', round(e['value'],1), 'wall_ms', round(e.get('wall_s',0)*1000,2), 'init', e.get('init_ms'), e.get('init_phases_ms'), 'loop', e.get('loop_ms'))"
  done
done
