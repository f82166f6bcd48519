# claim-batch sweep of the generation kernel (GSGP_GSM_BATCH; 0 = automatic)
rm -f gpurun_out/gsm_batch.log
for b in ${BATCHES:-0 8 16 32 64}; do
  for c in ${AB_CFGS:-c3 c4s c5 c2}; do
    r=$(GSGP_GSM_BATCH=$b timeout 600 python bench.py --config $c --steps ${AB_STEPS:-30} --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
    echo "batch=$b $c $r" | tee -a gpurun_out/gsm_batch.log
  done
done
