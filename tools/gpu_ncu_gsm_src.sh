# ncu --set full with source of one GSM launch (C4-shaped and C3-shaped), plus short C4/C3 bench lines
set -x
O=gpurun_out/${OUT:-r02/ncu_gsm_src}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o $O/prof_gsm_c4s \
  python bench.py --config c4s --steps 8 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_c4s.log 2>&1; echo "rc=$?"
timeout 600 python bench.py --config c4 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
cat $O/bench_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks'])"
