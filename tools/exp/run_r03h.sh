#!/usr/bin/env bash
set -u
o=gpurun_out/r03h; mkdir -p $o
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dt_tmem" -c 2 \
    -o $o/tmem python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
