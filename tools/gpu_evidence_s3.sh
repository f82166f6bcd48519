# Final round-2 evidence with the final kernels: GPU suite + smoke, default bench, reference arm,
# C2/C4/C5 lines, ncu launch list of the default command, ncu full captures (C2 engine kernels),
# C3 GSM DRAM bytes per launch.
set -x
O=gpurun_out/r02/${EV:-ev3}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/gpu_info.csv
lscpu | grep -E "Model name|^CPU\(s\)" > $O/cpu_info.txt
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
for c in c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv \
  python bench.py > $O/ncu_launch_default.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o $O/prof_gsm_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_gsm_c2.log 2>&1; echo "gsm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o $O/prof_interp_c2 \
  python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_interp_c2.log 2>&1; echo "interp rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_survive -s 5 -c 1 -o $O/prof_survive_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_survive_c2.log 2>&1; echo "survive rc=$?"
timeout 1200 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:k_gsm_tma -s 3 -c 1 --csv --log-file $O/ncu_c3_gsm_dram.csv \
  python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_c3.log 2>&1; echo "c3 dram rc=$?"
tail -n 3 $O/*.err
