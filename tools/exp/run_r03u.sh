#!/usr/bin/env bash
set -u
o=gpurun_out/r03u; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "build_pdm_set or precompute or distance or config or golden or tile_bounds or flags_merge or packed" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_$r.json 2>&1; echo "pre rc=$?" >> $o/status.txt
done
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dt_tmem" -c 2 \
    -o $o/tmem python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
