# bench lines for the default (C3) run and the other BASELINE configs
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in ${BENCH_CFGS:-c4 c5}; do
  timeout 900 python bench.py --config $c --steps ${BENCH_STEPS:-50} --no-cpu-baseline --no-secondary > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
tail -c 600 gpurun_out/bench_default.json
