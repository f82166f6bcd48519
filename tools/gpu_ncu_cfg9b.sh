set -x
O=gpurun_out/r02/ncu_cfg9b; mkdir -p $O
GSGP_INTERP_CFG=9 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o $O/prof_interp_c2_cfg9u2 \
  python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu.log 2>&1; echo "rc=$?"
