# same-box A/B of library variants on the generation loop.  Variants
# (ABVARS, order rotated every repetition: the box is power-capped):
#   old      ab_old/bench.py (a previous commit's package, built)
#   new      the working tree
#   lib:X    the working tree with GSGP_LIB=ab/X.so
for rep in 1 2 3; do
  set -- ${ABVARS:-old new}
  vars="$*"
  if [ $((rep % 2)) = 0 ]; then vars=$(echo $vars | tr ' ' '\n' | tac | tr '\n' ' '); fi
  for v in $vars; do
    for c in ${ABCFGS:-c2 c3}; do
      case $v in
        old) cmd="python ab_old/bench.py";;
        new) cmd="python bench.py";;
        lib:*) cmd="env GSGP_LIB=ab/${v#lib:}.so python bench.py";;
      esac
      timeout 600 $cmd --config $c --steps ${ABSTEPS:-30} --warmup 5 --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 > gpurun_out/abv.json
      python -c "
import json; d=json.load(open('gpurun_out/abv.json')); r=d['roofline']
print('$rep $v $c', round(d['value'],2), 'step', round(d['ms_per_step'],5), 'gsm', round(r['avg_launch_ms'],5), 'other_us', round((d['ms_per_step']-r['avg_launch_ms'])*1000,1), d['clocks']['sm_mhz'])"
    done
  done
done
