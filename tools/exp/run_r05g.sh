#!/usr/bin/env bash
# 256^3 acceptance case: raw planes for every k (PDM_RAW_MAX_K=64) vs packed above k=4
set -u
o=gpurun_out/r05g; mkdir -p $o
for r in 1 2; do
for kk in 4 64; do
PDM_RAW_MAX_K=$kk timeout 300 python tools/exp/small_update_probe.py > $o/small_$kk.$r.json 2>>$o/err.txt; echo "small $kk rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
