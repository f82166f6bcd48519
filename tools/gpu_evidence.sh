# Round evidence: default bench, reference arm, ncu launch list of the default command,
# full ncu captures of the three engine kernels at C2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu_info.csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/cpu_info.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
  python bench.py > gpurun_out/ncu_launch_default.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o gpurun_out/prof_gsm_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gsm_c2.log 2>&1; echo "gsm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o gpurun_out/prof_interp_c2 \
  python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_interp_c2.log 2>&1; echo "interp rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_survive -s 5 -c 1 -o gpurun_out/prof_survive_c2 \
  python bench.py --config c2 --steps 10 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_survive_c2.log 2>&1; echo "survive rc=$?"
cat gpurun_out/bench_default.json; cat gpurun_out/bench_reference.json; tail -n 3 gpurun_out/*.err
