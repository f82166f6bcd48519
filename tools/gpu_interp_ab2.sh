# interpreter: parity tests of the in-tree lib, then A/B vs gsm_alt/*.so (init only, 2 reps)
set -x
O=gpurun_out/${AB_OUT:-r02/interp}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_headline_paths.py tests/test_gpu_run.py tests/test_gpu_random_runs.py -q -m gpu -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for rep in 1 2; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  for c in ${SHAPES:-c2 c3 c5 c4}; do
   echo "$rep lib=$lib $(GSGP_LIB=$PWD/$lib timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a $O/ab.log
  done
done
done
