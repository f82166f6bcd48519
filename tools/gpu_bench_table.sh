# bench lines for every BASELINE config (GSM table in DESIGN.md §6)
mkdir -p gpurun_out/tab
timeout 900 python bench.py --no-secondary > gpurun_out/tab/c3.json 2> gpurun_out/tab/c3.err
timeout 600 python bench.py --config c2 --steps 500 --no-cpu-baseline --no-secondary > gpurun_out/tab/c2.json 2> gpurun_out/tab/c2.err
timeout 600 python bench.py --config c1 --steps 50 --no-cpu-baseline --no-secondary > gpurun_out/tab/c1.json 2> gpurun_out/tab/c1.err
timeout 900 python bench.py --config c4 --steps 50 --no-cpu-baseline --no-secondary > gpurun_out/tab/c4.json 2> gpurun_out/tab/c4.err
timeout 900 python bench.py --config c5 --steps 50 --no-cpu-baseline --no-secondary > gpurun_out/tab/c5.json 2> gpurun_out/tab/c5.err
for c in c1 c2 c3 c4 c5; do python -c "
import json; d=json.loads(open('gpurun_out/tab/$c.json').read().strip().splitlines()[-1]); r=d['roofline']; e=d['e2e'] or {}
print('$c', round(d['value'],2), round(r['achieved']), round(r['frac'],4), 'e2e', e.get('value') and round(e['value'],2), 'init', round(d['init_ms']['compute_semantics']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
