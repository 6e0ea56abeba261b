#!/usr/bin/env bash
set -u
o=gpurun_out/r04z; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "distance or precompute or build_pdm_set or tile_bounds or random_volumes or at_size or standard" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do timeout 300 python tools/precompute_bench.py > $o/pre_$r.json 2>&1; done
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none -k "regex:dt_tmem" -c 1 -o $o/tmem python tools/exp/precompute_once.py 1 > $o/ncu.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
