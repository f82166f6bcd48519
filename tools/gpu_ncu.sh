# ncu evidence for profiles/: launch list (cold, serialised) + full capture of the top kernels
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm -s 3 -c 2 -o gpurun_out/prof_gsm_c2 \
  python bench.py --config c2 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gsm.log 2>&1; echo "gsm full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 2 -o gpurun_out/prof_interp_c2 \
  python bench.py --config c2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_interp.log 2>&1; echo "interp full rc=$?"
ls -la gpurun_out
