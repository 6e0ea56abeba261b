#!/usr/bin/env bash
set -u
o=gpurun_out/r02p; mkdir -p $o
python tools/exp/merge_once.py > $o/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:combine_packed_flags -c 3 -o $o/merge_skip python tools/exp/merge_once.py > $o/ncu_skip.log 2>&1
echo "ncu skip rc=$?" >> $o/status.txt
PDM_TILE_SKIP=0 python tools/exp/merge_once.py > $o/plain2.log 2>&1 && \
PDM_TILE_SKIP=0 ncu --set full --clock-control none --import-source on -k regex:combine_packed_flags -c 3 -o $o/merge_noskip python tools/exp/merge_once.py > $o/ncu_noskip.log 2>&1
echo "ncu noskip rc=$?" >> $o/status.txt
