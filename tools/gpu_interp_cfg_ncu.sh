# interpreter launch-config A/B by ncu kernel duration (GSGP_INTERP_CFG)
rm -f gpurun_out/interp_cfg_ncu.log
for cfg in ${CFGS:-0 1}; do
  for c in ${SHAPES:-c2}; do
    GSGP_INTERP_CFG=$cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_interpret --csv \
      python tools/probe_interp.py $c 1 2>/dev/null | grep k_interpret | awk -F'","' -v cfg=$cfg -v c=$c '{gsub(/"/,"",$NF); print "cfg="cfg, c, $5, $NF}' >> gpurun_out/interp_cfg_ncu.log
  done
done
cat gpurun_out/interp_cfg_ncu.log
