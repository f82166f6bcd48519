# interpreter cfg 10 program-loop unroll A/B (gsm_alt/unroll{2,3,4}.so), alternating, 2 reps
set -x
O=gpurun_out/${AB_OUT:-r02/ab_unroll10}; mkdir -p $O
for rep in 1 2; do
for lib in gsm_alt/unroll4.so gsm_alt/unroll2.so gsm_alt/unroll3.so; do
  for c in c2 c3 c4; do
    echo "$rep $lib $c $(GSGP_LIB=$PWD/$lib timeout 600 python tools/probe_interp.py $c 2 2>/dev/null)" | cut -c1-160 | tee -a $O/ab.log
  done
done
done
timeout 600 python -m pytest tests/test_gpu_op_mix.py -q -p no:cacheprovider > $O/pytest_op_mix.log 2>&1; echo "op mix rc=$?"; tail -3 $O/pytest_op_mix.log
