#!/usr/bin/env bash
set -u
o=gpurun_out/r03k; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_m6_$r.json 2>&1; echo "m6 rc=$?" >> $o/status.txt
for v in m7 m8 m7r3; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 300 python tools/precompute_bench.py > $o/pre_${v}_$r.json 2>&1; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
