mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm -s 3 -c 1 -o gpurun_out/prof_gsm_tma_c2 \
  python bench.py --config c2 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gsm_tma.log 2>&1; echo "rc=$?"
GSGP_GSM_LEGACY=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm -s 3 -c 1 -o gpurun_out/prof_gsm_legacy_c2 \
  python bench.py --config c2 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gsm_legacy.log 2>&1; echo "rc=$?"
