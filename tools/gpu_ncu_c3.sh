mkdir -p gpurun_out
timeout 1200 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum -k regex:k_gsm_tma -s 3 -c 1 --csv --log-file gpurun_out/ncu_c3_dram.csv \
  python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "rc=$?"
cat gpurun_out/ncu_c3_dram.csv | tail -8
