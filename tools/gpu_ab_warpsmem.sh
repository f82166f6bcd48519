# one-warp genome groups: shared-memory cap 220 vs 226 KB (gsm_alt/ring220.so vs ring226.so)
set -x
O=gpurun_out/${AB_OUT:-r02/ab_warpsmem}; mkdir -p $O
for rep in 1 2; do
for lib in gsm_alt/ring220.so gsm_alt/ring226.so; do
  for c in c5 c5s; do
    echo "$rep $lib $c $(GSGP_LIB=$PWD/$lib GSGP_INTERP_TRACE=1 timeout 600 python tools/probe_interp.py $c 2 2>>$O/trace_$(basename $lib).log)" | cut -c1-200 | tee -a $O/ab.log
  done
done
done
