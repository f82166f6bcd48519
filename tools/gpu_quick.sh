mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for cfgname in ${CONFIGS:-c2 c3}; do
  st=200; [ $cfgname = c3 ] && st=50
  timeout 900 python bench.py --config $cfgname --steps $st --warmup 5 --no-cpu-baseline ${BENCH_EXTRA} > gpurun_out/bench_${cfgname}.json 2> gpurun_out/bench_${cfgname}.err; echo "bench $cfgname rc=$?"; tail -n 3 gpurun_out/bench_${cfgname}.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_c*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d['roofline']; e=d.get('e2e') or {}
        print(f, round(d['value'],2), 'gen/s', round(r['achieved'],1), 'GB/s', round(r['frac'],3), 'share', round(r['kernel_share_of_step'],3), 'e2e', round(e.get('value',0),2), 'init', d['init_ms'], 'e2e_init', e.get('init_ms'))
    except Exception as ex: print(f, 'ERR', ex)
PY
