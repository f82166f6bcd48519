python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider 2>&1 | tail -2
for c in ${CONFIGS:-c4s c2 c3 c4}; do st=100; [ $c = c3 ] && st=50; python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
python - <<PY
import json, os
for c in os.environ.get("CONFIGS", "c4s c2 c3 c4").split():
    try:
        d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1]); r=d["roofline"]
        print(c, round(d["value"],2), round(r["achieved"],1), round(r["frac"],3), round(r["kernel_share_of_step"],3))
    except Exception as e: print(c, "ERR", e, open(f"gpurun_out/bench_{c}.err").read()[-300:])
PY
