set -x
O=gpurun_out/r02/ncu_c5; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o $O/prof_interp_c5s \
  python bench.py --config c5s --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu.log 2>&1; echo "rc=$?"
