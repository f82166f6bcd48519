# sustained C3: 1000 timed generations (~22 s at the board power cap), clocks sampled throughout
set -x
O=gpurun_out/r02/sustained; mkdir -p $O
timeout 900 python bench.py --config c3 --steps 1000 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $O/bench_c3_1000.json 2> $O/bench_c3_1000.err; echo "rc=$?"
python -c "import json; d=json.load(open('$O/bench_c3_1000.json')); print(round(d['value'],2), round(d['roofline']['frac'],4), d['clocks'])"
