set -x
O=gpurun_out/r02/final_check; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; cat $O/smoke.log
timeout 300 python tools/probe_interp.py c2 2 > $O/probe_c2.json 2>&1; cat $O/probe_c2.json | cut -c1-200
