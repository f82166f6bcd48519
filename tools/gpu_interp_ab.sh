# interpreter A/B: in-tree library vs the builds in gsm_alt/ (GSGP_LIB), C2/C3/C5 init
rm -f gpurun_out/interp_ab.log
for rep in 1 2; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  for c in ${SHAPES:-c2 c3 c5}; do
   echo "lib=$lib $(GSGP_LIB=$PWD/$lib timeout 300 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a gpurun_out/interp_ab.log
  done
done
done
