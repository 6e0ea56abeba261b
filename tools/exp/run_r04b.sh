#!/usr/bin/env bash
# apron item order: x-chunk slowest vs the round-2 order
set -u
o=gpurun_out/r04b; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "apron or min_max or range_apron or random_volumes" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for side in 2048 1024; do
for r in 1 2; do
timeout 600 python tools/exp/apron_time.py $side > $o/new_${side}_$r.txt 2>&1; echo "new $side rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_rowmajor.so timeout 600 python tools/exp/apron_time.py $side > $o/old_${side}_$r.txt 2>&1; echo "old $side rc=$?" >> $o/status.txt
PDM_APRON_TMA=0 timeout 600 python tools/exp/apron_time.py $side > $o/cpa_${side}_$r.txt 2>&1; echo "cpa $side rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
