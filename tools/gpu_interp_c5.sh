# C5 interpreter A/B (global-feature prefetch): in-tree vs gsm_alt/base.so, plus parity tests
set -x
O=gpurun_out/r02/c5pf; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_run.py -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for rep in 1 2; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/base.so; do
  for c in c5 c5s; do
   echo "$rep lib=$lib $(GSGP_LIB=$PWD/$lib timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a $O/ab.log
  done
  echo "$rep lib=$lib forced-cfg2-c2 $(GSGP_INTERP_CFG=2 GSGP_LIB=$PWD/$lib timeout 300 python tools/probe_interp.py c2 2 2>&1 | tail -1)" | tee -a $O/ab.log
done
done
