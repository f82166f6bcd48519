# full GPU suite + C5 and C3 bench lines
set -x
O=gpurun_out/${OUT:-r02/check2}; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
timeout 400 python bench.py --config c5 --steps 50 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
timeout 400 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python -c "
import json
for c in ('c5','c3'):
    d=json.load(open('$O/bench_'+c+'.json')); print(c, round(d['value'],2), round(d['roofline']['frac'],4), d['e2e']['value'], d['interpreter']['seconds'], d['interpreter']['node_evals_per_s'], d['interpreter']['fp64_roofline']['frac'])"
