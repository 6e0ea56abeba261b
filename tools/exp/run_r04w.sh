#!/usr/bin/env bash
# x pass from the mask: columns claimed dynamically vs static
set -u
o=gpurun_out/r04w; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "build_pdm_set or random_volumes or precompute or tile_bounds" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_dyn_$r.json 2>&1; echo "dyn rc=$?" >> $o/status.txt
PDM_XMASK_STATIC=1 timeout 300 python tools/precompute_bench.py > $o/pre_static_$r.json 2>&1; echo "static rc=$?" >> $o/status.txt
done
cat $o/status.txt
