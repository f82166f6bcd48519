set -x
O=gpurun_out/r02/padclear; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 600 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline --no-secondary > $O/bench_c3.json 2>/dev/null
python -c "import json; d=json.load(open('$O/bench_c3.json')); print('c3', round(d['value'],2), d['e2e']['value'], d['e2e']['init_ms'], d['e2e']['init_phases_ms'])"
