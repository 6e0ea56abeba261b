#!/usr/bin/env bash
# apron TMA ring depth A/B
set -u
o=gpurun_out/r03w; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
PDM_LIB_PATH=$V/libpdm_b200_r3.so timeout 900 python -m pytest tests -m gpu -q -x -k "apron or min_max or range_apron" > $o/pytest_r3.txt 2>&1; echo "pytest r3 rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_r2_$r.json 2>&1; echo "r2 rc=$?" >> $o/status.txt
for v in r3 r4; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 300 python tools/precompute_bench.py > $o/pre_${v}_$r.json 2>&1; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
