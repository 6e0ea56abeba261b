#!/usr/bin/env bash
set -u
o=gpurun_out/r02v; mkdir -p $o
python tools/exp/precompute_once.py 1 > $o/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:apron_fast|dt_tile|dt_dist1d|dt_expand|tile_bounds" -c 6 -o $o/pre python tools/exp/precompute_once.py 1 > $o/ncu.log 2>&1
echo "ncu rc=$?" >> $o/status.txt
