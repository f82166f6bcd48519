# SM clock / power while the C3 interpreter runs (NVML sampling every 20 ms)
set -x
O=gpurun_out/r02/interp_clock; mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 20 > $O/smi.csv &
SMI=$!
sleep 1
timeout 600 python tools/probe_interp.py c3 3 > $O/probe_c3.json 2> $O/probe_c3.err; echo "probe rc=$?"
kill $SMI
cat $O/probe_c3.json | cut -c1-200
python - <<'PY'
import csv, statistics
rows=[r for r in csv.reader(open('gpurun_out/r02/interp_clock/smi.csv'))]
clk=[float(r[1].split()[0]) for r in rows if 'MHz' in r[1]]
pw=[float(r[2].split()[0]) for r in rows if 'W' in r[2]]
busy=[(c,p) for c,p in zip(clk,pw) if p>300]
print('samples', len(clk), 'busy', len(busy))
if busy:
    print('median clock under load', statistics.median([c for c,_ in busy]), 'median power', statistics.median([p for _,p in busy]), 'max power', max(p for _,p in busy))
PY
