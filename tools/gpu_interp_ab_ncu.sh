# interpreter A/B by kernel duration (ncu launch list), in-tree lib vs gsm_alt/*.so
rm -f gpurun_out/interp_ab_ncu.log
for rep in 1 2 3; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/*.so; do
  for c in ${SHAPES:-c2 c5s}; do
    GSGP_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_interpret --csv \
      python tools/probe_interp.py $c 1 2>/dev/null | grep k_interpret | awk -F'","' -v lib=$lib -v c=$c '{gsub(/"/,"",$NF); print lib, c, $5, $NF}' >> gpurun_out/interp_ab_ncu.log
  done
done
done
cat gpurun_out/interp_ab_ncu.log
