# interpreter launch configurations forced by GSGP_INTERP_CFG (init only), C2/C3/C4
set -x
O=gpurun_out/${AB_OUT:-r02/interp_cfg}; mkdir -p $O
for rep in 1 2; do
for cfg in ${CFGS:-7 9 10 1}; do
  for c in ${SHAPES:-c2 c3 c4}; do
   echo "$rep cfg=$cfg $(GSGP_INTERP_CFG=$cfg timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a $O/ab.log
  done
done
done
