set -x
O=gpurun_out/r02/scaling; mkdir -p $O
timeout 1200 python tools/probe_scaling.py 40 > $O/probe_scaling.jsonl 2> $O/probe_scaling.err; echo "rc=$?"; cat $O/probe_scaling.jsonl; tail -3 $O/probe_scaling.err
