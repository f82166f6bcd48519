# Reference arm beside our arm on every BASELINE config (C1/C2 at full size, C3-C5 on bounded samples)
set -x
O=gpurun_out/r02/ref_table; mkdir -p $O
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --impl reference --steps 5 --warmup 3 > $O/ref_$c.json 2> $O/ref_$c.err; echo "ref $c rc=$?"
done
for c in ${OURS:-c1 c2}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-secondary > $O/ours_$c.json 2> $O/ours_$c.err; echo "ours $c rc=$?"
done
