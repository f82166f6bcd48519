# ncu --set full with source of the C5-shaped interpreter launch (one-warp genome groups, cfg 9)
set -x
O=gpurun_out/${OUT:-r02/ncu_c5s_interp}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o $O/prof_interp_c5s \
  python tools/probe_interp.py c5s 1 > $O/ncu.log 2>&1; echo "rc=$?"
tail -2 $O/ncu.log
