# interpreter A/B by ncu kernel duration over environment settings (ENVS="A=1 A=0")
rm -f gpurun_out/interp_env_ab.log
for rep in 1 2; do
for e in ${ENVS:-GSGP_INTERP_THREADED=1 GSGP_INTERP_THREADED=0}; do
  for c in ${SHAPES:-c2}; do
    env $e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_interpret --csv \
      python tools/probe_interp.py $c 1 2>/dev/null | grep k_interpret | awk -F'","' -v e=$e -v c=$c '{gsub(/"/,"",$NF); print e, c, $NF}' >> gpurun_out/interp_env_ab.log
  done
done
done
cat gpurun_out/interp_env_ab.log
