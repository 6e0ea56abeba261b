#!/usr/bin/env bash
# A/B: sweep word packing by folded shift-adds (variant pk) vs current
set -u
o=gpurun_out/r05b; mkdir -p $o
V=paper_2407_21552_b200/lib/variants/libpdm_b200_pk.so
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_base$r.json 2>>$o/err.txt; echo "base rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V timeout 300 python tools/precompute_bench.py > $o/pre_pk$r.json 2>>$o/err.txt; echo "pk rc=$?" >> $o/status.txt
done
PDM_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dt or distance or pdm_set or standard or tmem or sweep" > $o/parity.txt 2>&1; echo "parity rc=$?" >> $o/status.txt
cat $o/status.txt
