# A/B of generation-kernel variants (GSGP_LIB builds in gsm_alt/)
rm -f gpurun_out/gsm_ab.log
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  for c in ${AB_CFGS:-c4s c2 c5}; do
    r=$(GSGP_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps ${AB_STEPS:-30} --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
    echo "$lib $c $r" | tee -a gpurun_out/gsm_ab.log
  done
done
