# interpreter A/B of library builds (GSGP_LIB) on the C2/C3 init: IAVARS = "default lib_x ..."
for rep in 1 2; do
  for v in ${IAVARS:-default}; do
    for c in c2 c3; do
      if [ $v = default ]; then L=""; else L="GSGP_LIB=ab/$v.so"; fi
      echo "rep $rep $v $(env $L timeout 600 python tools/probe_interp.py $c 2 2>&1 | tail -1)"
    done
  done
done
