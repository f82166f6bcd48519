mkdir -p gpurun_out
timeout 1200 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:k_gsm_tma -s 3 -c 1 --csv --log-file gpurun_out/ncu_c4.csv \
  python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
grep -o '"[a-z_.]*","[%a-z]*","[0-9.]*"' gpurun_out/ncu_c4.csv
