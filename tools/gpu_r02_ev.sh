# Round-2 evidence: default bench, reference arm, ncu launch list of the default command,
# full ncu captures of GSM / interpreter / reduce-survive at C2, C3 GSM DRAM traffic,
# C4/C5 bench lines, tail probe.
set -x
E=gpurun_out/${EV:-r02/ev}
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $E/gpu_info.csv
lscpu | grep -E "Model name|^CPU\(s\)" > $E/cpu_info.txt
timeout 900 python bench.py > $E/bench_default.json 2> $E/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $E/bench_reference.json 2> $E/bench_reference.err; echo "ref rc=$?"
timeout 600 python tools/probe_tail.py c2 200 > $E/probe_tail_c2.jsonl 2> $E/probe_tail_c2.err; echo "tail rc=$?"
for c in c4 c5; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --no-secondary > $E/bench_$c.json 2> $E/bench_$c.err; echo "$c rc=$?"
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_default.csv \
  python bench.py > $E/ncu_launch_default.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o $E/prof_gsm_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $E/ncu_gsm_c2.log 2>&1; echo "gsm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o $E/prof_interp_c2 \
  python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $E/ncu_interp_c2.log 2>&1; echo "interp rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_survive -s 5 -c 1 -o $E/prof_survive_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $E/ncu_survive_c2.log 2>&1; echo "survive rc=$?"
timeout 1200 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:k_gsm_tma -s 3 -c 1 --csv --log-file $E/ncu_c3_gsm_dram.csv \
  python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $E/ncu_c3.log 2>&1; echo "c3 dram rc=$?"
cat $E/bench_default.json; cat $E/bench_reference.json; cat $E/probe_tail_c2.jsonl; tail -n 3 $E/*.err
