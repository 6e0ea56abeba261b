#!/usr/bin/env bash
# A/B: x pass from the mask with one CTA of 16 / 20 / 24 warps per SM vs 2 x 8
set -u
o=gpurun_out/r05e; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_base$r.json 2>>$o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in x16 x20 x24; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 300 python tools/precompute_bench.py > $o/pre_$v$r.json 2>>$o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
PDM_LIB_PATH=$V/libpdm_b200_x24.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $o/parity24.txt 2>&1; echo "parity24 rc=$?" >> $o/status.txt
cat $o/status.txt
