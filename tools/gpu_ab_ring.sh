# interpreter A/B: program ring for one-warp genome groups (in-tree) vs the previous library (gsm_alt/base.so)
set -x
O=gpurun_out/${AB_OUT:-r02/ab_ring}; mkdir -p $O
for rep in 1 2; do
for lib in gsm_alt/base.so paper_2106_04034_b200/libgsgp_b200.so; do
  for c in c5 c5s; do
    echo "$rep $lib $c $(GSGP_LIB=$PWD/$lib GSGP_INTERP_TRACE=1 timeout 600 python tools/probe_interp.py $c 2 2>>$O/trace.log)" | tee -a $O/ab.log
  done
  for c in c2 c3; do
    echo "$rep $lib cfg9 $c $(GSGP_LIB=$PWD/$lib GSGP_INTERP_CFG=9 timeout 600 python tools/probe_interp.py $c 2 2>/dev/null)" | tee -a $O/ab.log
  done
done
done
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -k "interp or semantics or golden or run" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
