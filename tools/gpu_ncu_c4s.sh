mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o gpurun_out/prof_gsm_c4s \
  python bench.py --config c4s --steps 8 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gsm_c4s.log 2>&1; echo "rc=$?"
timeout 600 python bench.py --config c4s --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4s.json 2>&1; echo "bench rc=$?"
