#!/usr/bin/env bash
# full captures (source-level) of the merge at k=16 and the precompute kernels
set -u
o=gpurun_out/r03e; mkdir -p $o
python tools/exp/merge_once.py 16 > $o/m_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:combine_packed_flags -c 1 \
    -o $o/merge_k16 python tools/exp/merge_once.py 16 > $o/ncu_m.log 2>&1; echo "ncu merge rc=$?" >> $o/status.txt
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k "regex:apron_fast|dt_tile|dt_dist1d|dt_expand" -c 5 \
    -o $o/pre python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu pre rc=$?" >> $o/status.txt
cat $o/status.txt
