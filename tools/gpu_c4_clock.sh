# C4 steady-state: long loops so the clock samples are dominated by the GSM loop; c4s beside it; c2 line for the interpreter rooflines
set -x
O=gpurun_out/${OUT:-r02/c4_clock}; mkdir -p $O
for c in c4 c4s c2; do
  st=200; [ $c = c4s ] && st=1000; [ $c = c2 ] && st=300
  timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
  python -c "import json; d=json.load(open('$O/bench_$c.json')); print('$c', round(d['value'],2), round(d['roofline']['frac'],4), d['clocks']); print(json.dumps(d['interpreter']))"
done
