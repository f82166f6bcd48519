# full GPU suite + short C2/C3 bench lines
set -x
O=gpurun_out/${OUT:-r02/check}; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
timeout 300 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline --no-secondary > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json
for c in ('c2','c3'):
    d=json.load(open('$O/bench_'+c+'.json')); print(c, round(d['value'],2), round(d['roofline']['frac'],4), d['e2e']['value'], json.dumps(d['interpreter']))"
