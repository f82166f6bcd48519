# round 2: full gpu suite, interpreter A/B (register-feature vs grouped smem), fp64 peak
set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r02a/fp64_peak.json; cat gpurun_out/r02a/fp64_peak.json
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r02a/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02a/pytest_gpu.log
for c in c2 c3; do
  for v in rf norf; do
    if [ $v = norf ]; then export GSGP_INTERP_NO_RF=1; else unset GSGP_INTERP_NO_RF; fi
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/r02a/bench_${c}_$v.json 2> gpurun_out/r02a/bench_${c}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/r02a/bench_${c}_$v.json'));print('$c $v', d['init_ms'], d['value'])"
  done
done
unset GSGP_INTERP_NO_RF
