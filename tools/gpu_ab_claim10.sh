# interpreter grouped blocks: static round-robin genomes per group vs dynamic block-local claiming
set -x
O=gpurun_out/${AB_OUT:-r02/ab_claim10}; mkdir -p $O
for rep in 1 2; do
for lib in gsm_alt/static.so gsm_alt/dynamic.so; do
  for c in c2 c3 c4; do
    echo "$rep $lib $c $(GSGP_LIB=$PWD/$lib timeout 600 python tools/probe_interp.py $c 2 2>/dev/null)" | sed -E 's/"compute_semantics_ms": \[[^]]*\], //' | cut -c1-150 | tee -a $O/ab.log
  done
done
done
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -k "interp or semantics or golden or run or op_mix or headline" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
