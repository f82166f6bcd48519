# quick generation-kernel + init check: gpu tests, then c3 (30 steps), c4s, c5, c2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in ${QCFGS:-c3 c4s c5 c2}; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-secondary $QARGS 2>/dev/null | tail -1 > gpurun_out/q_$c.json
  python -c "
import json; d=json.load(open('gpurun_out/q_$c.json')); e=d['e2e'] or {}
print('$c', round(d['value'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], 'e2e', e.get('value') and round(e['value'],2), e.get('init_ms') and round(e['init_ms']), e.get('init_phases_ms'))"
done
