# interpreter A/B: 128x3 single-genome blocks (cfg 5) vs two genome groups per block (cfg 6), C2 and C3 init
for rep in 1 2; do
  for cfg in 5 6; do
    for c in c2 c3; do
      echo "rep $rep cfg $cfg $(GSGP_INTERP_CFG=$cfg timeout 600 python tools/probe_interp.py $c 2 2>&1 | tail -1)"
    done
  done
done
GSGP_INTERP_CFG=6 timeout 600 python tools/probe_interp_occupancy.py 400000
