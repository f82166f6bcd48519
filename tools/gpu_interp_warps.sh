# one-warp genome groups (cfg 9): parity, then A/B vs the default configuration
set -x
O=gpurun_out/r02/warps; mkdir -p $O
timeout 420 python -m pytest tests/test_gpu_ops.py tests/test_gpu_random_runs.py -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for rep in 1 2; do
for cfg in ${CFGS:-default 9}; do
  for c in c2 c3 c4 c5; do
   if [ $cfg = default ]; then unset GSGP_INTERP_CFG; else export GSGP_INTERP_CFG=$cfg; fi
   echo "$rep cfg=$cfg $(timeout 120 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a $O/ab.log
  done
done
done
unset GSGP_INTERP_CFG
