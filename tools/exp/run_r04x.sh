#!/usr/bin/env bash
# apron: items claimed dynamically vs static
set -u
o=gpurun_out/r04x; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_dyn_$r.json 2>&1; echo "dyn rc=$?" >> $o/status.txt
PDM_APRON_STATIC=1 timeout 300 python tools/precompute_bench.py > $o/pre_static_$r.json 2>&1; echo "static rc=$?" >> $o/status.txt
done
timeout 600 python tools/exp/apron_time.py 2048 > $o/d_dyn.txt 2>&1
PDM_APRON_STATIC=1 timeout 600 python tools/exp/apron_time.py 2048 > $o/d_static.txt 2>&1
cat $o/status.txt
