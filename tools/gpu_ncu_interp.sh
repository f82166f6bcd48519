# ncu --set full of the interpreter (population mode, C2 init) with source, per config
set -x
mkdir -p gpurun_out
for cfg in ${CFGS:-0}; do
GSGP_INTERP_CFG=$cfg timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_interpret -c 1 -o gpurun_out/prof_interp_c2_cfg$cfg \
  python tools/probe_interp.py c2 1 > gpurun_out/ncu_interp_cfg$cfg.log 2>&1; echo "interp full rc=$?"
done
ls -la gpurun_out
