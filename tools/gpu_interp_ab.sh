rm -f gpurun_out/interp_ab.log
for lib in paper_2106_04034_b200/libgsgp_b200.so tools/alt/libgsgp_b200_unroll1.so; do
 for cfg in 0 6; do
  for c in c2 c3; do
   echo "lib=$lib cfg=$cfg $(GSGP_LIB=$PWD/$lib GSGP_INTERP_CFG=$cfg timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a gpurun_out/interp_ab.log
  done
 done
done
