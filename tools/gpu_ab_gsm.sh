# GSM A/B: in-tree library vs gsm_alt/*.so (alternating, 2 reps), then the full GPU suite on the in-tree lib
set -x
O=gpurun_out/${AB_OUT:-r02/ab}; mkdir -p $O
for rep in 1 2; do
for lib in gsm_alt/*.so paper_2106_04034_b200/libgsgp_b200.so; do
  for c in ${AB_CFGS:-c4s c4 c2 c3 c5}; do
    st=30; [ $c = c2 ] && st=300; [ $c = c4s ] && st=100
    r=$(GSGP_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))")
    echo "$rep $lib $c $r" | tee -a $O/ab.log
  done
done
done
if [ -z "$AB_NO_TESTS" ]; then
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
fi
