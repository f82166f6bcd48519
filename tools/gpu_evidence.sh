# Round evidence: default bench, reference arm, ncu launch list of the default command,
# full ncu captures of the three engine kernels at C2, C3 GSM DRAM traffic per launch.
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/ev/gpu_info.csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/ev/cpu_info.txt
timeout 900 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_default.csv \
  python bench.py > gpurun_out/ev/ncu_launch_default.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o gpurun_out/ev/prof_gsm_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ev/ncu_gsm_c2.log 2>&1; echo "gsm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o gpurun_out/ev/prof_interp_c2 \
  python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ev/ncu_interp_c2.log 2>&1; echo "interp rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_survive -s 5 -c 1 -o gpurun_out/ev/prof_survive_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ev/ncu_survive_c2.log 2>&1; echo "survive rc=$?"
timeout 1200 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:k_gsm_tma -s 3 -c 1 --csv --log-file gpurun_out/ev/ncu_c3_gsm_dram.csv \
  python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/ev/ncu_c3.log 2>&1; echo "c3 dram rc=$?"
cat gpurun_out/ev/bench_default.json; cat gpurun_out/ev/bench_reference.json; tail -n 3 gpurun_out/ev/*.err
