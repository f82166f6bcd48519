# ncu --set full (with source/SASS stall sampling) of the default interpreter config, C2 population launch
set -x
O=gpurun_out/${OUT:-r02/ncu_interp_src}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o $O/prof_interp_c2 \
  python tools/probe_interp.py c2 1 > $O/ncu.log 2>&1; echo "rc=$?"
tail -3 $O/ncu.log
