# parity + interpreter throughput per launch configuration (GSGP_INTERP_CFG)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-auto 0 1 2 3 4 5}; do
  for c in ${SHAPES:-c2 c3 c5}; do
    if [ "$cfg" = auto ]; then unset GSGP_INTERP_CFG; else export GSGP_INTERP_CFG=$cfg; fi
    echo "cfg=$cfg $(timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a gpurun_out/interp_cfgs.log
  done
done
