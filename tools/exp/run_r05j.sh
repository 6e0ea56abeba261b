#!/usr/bin/env bash
# TMEM sweep shape for mid-size sets (config e n = 8, 16): auto vs forced one-CTA
set -u
o=gpurun_out/r05j; mkdir -p $o
for n in 8 16; do for r in 1 2; do
timeout 300 python tools/precompute_bench.py --n $n > $o/pre_n${n}_auto$r.json 2>>$o/err.txt; echo "n$n auto rc=$?" >> $o/status.txt
PDM_DT_TMEM_BIG=1 timeout 300 python tools/precompute_bench.py --n $n > $o/pre_n${n}_big$r.json 2>>$o/err.txt; echo "n$n big rc=$?" >> $o/status.txt
PDM_DT_TMEM_BIG=0 timeout 300 python tools/precompute_bench.py --n $n > $o/pre_n${n}_small$r.json 2>>$o/err.txt; echo "n$n small rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
