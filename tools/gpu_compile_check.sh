set -x
O=gpurun_out/r02/compile_smem; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -k "interp or semantics or golden or run or op_mix or compile or headline" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for c in c1 c2 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-secondary > $O/bench_$c.json 2>/dev/null; python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', round(d['value'],1), d['e2e']['value'], d['init_ms']['compile'], d['e2e']['init_phases_ms']['compile'])"; done
