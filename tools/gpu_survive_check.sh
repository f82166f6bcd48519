set -x
O=gpurun_out/r02/survive1pass; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for c in c1 c2 c3; do st=100; [ $c = c3 ] && st=30; timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline --no-secondary > $O/bench_$c.json 2>/dev/null; python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us/step', d['e2e']['value'])"; done
