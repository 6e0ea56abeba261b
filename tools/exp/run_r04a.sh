#!/usr/bin/env bash
# config d apron: x-run length and TMA vs cp.async
set -u
o=gpurun_out/r04a; mkdir -p $o
for xb in 32 8 128; do
PDM_APRON_XB=$xb timeout 600 python tools/exp/apron_time.py 2048 > $o/d_xb$xb.txt 2>&1; echo "xb$xb rc=$?" >> $o/status.txt
done
PDM_APRON_TMA=0 timeout 600 python tools/exp/apron_time.py 2048 > $o/d_cpa.txt 2>&1; echo "cpa rc=$?" >> $o/status.txt
for xb in 32 8; do
PDM_APRON_XB=$xb timeout 600 python tools/exp/apron_time.py 1024 > $o/c_xb$xb.txt 2>&1; echo "c xb$xb rc=$?" >> $o/status.txt
done
cat $o/status.txt
