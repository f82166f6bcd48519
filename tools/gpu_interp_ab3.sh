set -x
O=gpurun_out/r02/interp2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ops.py -q -m gpu -x -p no:cacheprovider -k "interp or division or semantics" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for f in gsm_alt/recip_u2.so gsm_alt/recip_u3.so; do GSGP_LIB=$PWD/$f timeout 900 python -m pytest tests/test_gpu_ops.py -q -m gpu -x -p no:cacheprovider -k "division" > $O/pytest_$(basename $f).log 2>&1; echo "pytest $f rc=$?"; done
for rep in 1 2; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  for c in c2 c3 c4; do
   echo "$rep lib=$lib $(GSGP_LIB=$PWD/$lib timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], d['interpret_pop_pool_ms'])")" | tee -a $O/ab.log
  done
done
done
