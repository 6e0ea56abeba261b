#!/usr/bin/env bash
set -u
o=gpurun_out/r03q; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "build_pdm_set or precompute or distance or config or golden or tile_bounds" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_new_$r.json 2>&1; echo "pre rc=$?" >> $o/status.txt
PDM_DT_XMASK=0 timeout 300 python tools/precompute_bench.py > $o/pre_old_$r.json 2>&1; echo "pre old rc=$?" >> $o/status.txt
done
cat $o/status.txt
