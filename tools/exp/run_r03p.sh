#!/usr/bin/env bash
set -u
o=gpurun_out/r03p; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_new_$r.json 2>&1; echo "pre rc=$?" >> $o/status.txt
PDM_DT_XMASK=0 timeout 300 python tools/precompute_bench.py > $o/pre_old_$r.json 2>&1; echo "pre old rc=$?" >> $o/status.txt
done
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dt_x_mask" -c 1 \
    -o $o/xmask python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
