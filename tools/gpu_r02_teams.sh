# GSM consumer teams A/B (gsm_alt/teams2.so vs in-tree), parity of the variant, ncu of C4s
set -x
O=gpurun_out/r02/teams; mkdir -p $O
GSGP_LIB=$PWD/gsm_alt/teams2.so timeout 900 python -m pytest tests/test_gpu_headline_paths.py tests/test_gpu_ops.py tests/test_gpu_run.py -q -m gpu -x -p no:cacheprovider > $O/pytest_teams2.log 2>&1; echo "pytest teams2 rc=$?"; tail -3 $O/pytest_teams2.log
for rep in 1 2; do
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/teams2.so; do
  for c in c4s c4 c2 c3 c5; do
    st=30; [ $c = c2 ] && st=300; [ $c = c4s ] && st=100
    r=$(GSGP_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-secondary 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms'],4), d['clocks']['sm_mhz'])")
    echo "$rep $lib $c $r" | tee -a $O/ab.log
  done
done
done
for lib in paper_2106_04034_b200/libgsgp_b200.so gsm_alt/teams2.so; do
  b=$(basename $lib .so)
  GSGP_LIB=$PWD/$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gsm_tma -s 5 -c 1 -o $O/prof_gsm_c4s_$b \
    python bench.py --config c4s --steps 8 --warmup 5 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_$b.log 2>&1; echo "ncu $b rc=$?"
done
