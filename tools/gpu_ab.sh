set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for cfgname in c2 c3; do
  st=200; [ $cfgname = c3 ] && st=50
  timeout 600 python bench.py --config $cfgname --steps $st --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfgname}_tma.json 2> gpurun_out/bench_${cfgname}_tma.err; echo "tma $cfgname rc=$?"
  GSGP_GSM_LEGACY=1 timeout 600 python bench.py --config $cfgname --steps $st --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfgname}_legacy.json 2> gpurun_out/bench_${cfgname}_legacy.err; echo "legacy $cfgname rc=$?"
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_*_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d['roofline']; print(f, round(d['value'],2), 'gen/s', round(r['achieved'],1), 'GB/s', round(r['frac'],3), 'share', round(r['kernel_share_of_step'],3), 'launch_ms', round(r['avg_launch_ms'],4))
    except Exception as e: print(f, 'ERR', e)
PY
for f in gpurun_out/*.err; do tail -n 3 $f; done
timeout 1200 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:k_gsm_tma -s 3 -c 1 --csv --log-file gpurun_out/ncu_c3_dram.csv \
  python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
grep -o '"dram__bytes[a-z_.]*","byte","[0-9]*"\|"lts__t_sector_hit_rate.pct","%","[0-9.]*"\|"gpu__time_duration.sum","[a-z]*","[0-9.]*"' gpurun_out/ncu_c3_dram.csv
