#!/usr/bin/env bash
# ncu of the merge at k=16 after the round-robin tile order (SM balance)
set -u
o=gpurun_out/r04r; mkdir -p $o
python tools/exp/merge_once.py 16 > $o/m_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:combine_packed_flags -c 1 \
    -o $o/merge_k16 python tools/exp/merge_once.py 16 > $o/ncu_m.log 2>&1; echo "ncu merge rc=$?" >> $o/status.txt
cat $o/status.txt
