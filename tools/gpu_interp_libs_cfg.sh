# interpreter A/B over libraries (in-tree + gsm_alt/*.so) with GSGP_INTERP_CFG=${ICFG:-9}, plus the in-tree default
set -x
O=gpurun_out/${AB_OUT:-r02/wunroll}; mkdir -p $O
for rep in 1 2; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  for c in ${SHAPES:-c2 c3 c5}; do
   echo "$rep lib=$lib cfg=${ICFG:-9} $(GSGP_INTERP_CFG=${ICFG:-9} GSGP_LIB=$PWD/$lib timeout 120 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a $O/ab.log
  done
done
done
for c in ${SHAPES:-c2 c3 c5}; do
  echo "0 lib=in-tree cfg=default $(timeout 120 python tools/probe_interp.py $c 2 2>&1 | tail -1)" | tee -a $O/ab.log
done
