#!/usr/bin/env bash
# A/B: TMEM sweep with one CTA of 28 (L=256) / 14 (L=512) warps per SM, or
# 24 / 12, vs 6 (3) CTAs of 4 warps
set -u
o=gpurun_out/r05c; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_base$r.json 2>>$o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in t28 t24; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 300 python tools/precompute_bench.py > $o/pre_$v$r.json 2>>$o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
timeout 600 python tools/precompute_bench.py --dims 2048 2048 2048 --reps 2 > $o/pre_d_base.json 2>>$o/err.txt; echo "d base rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_t28.so timeout 600 python tools/precompute_bench.py --dims 2048 2048 2048 --reps 2 > $o/pre_d_t28.json 2>>$o/err.txt; echo "d t28 rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_t28.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $o/parity.txt 2>&1; echo "parity rc=$?" >> $o/status.txt
cat $o/status.txt
