#!/usr/bin/env bash
# A/B: completion wait polling cudaStreamQuery (PDM_SPIN_US=200, default) vs
# blocking cudaStreamSynchronize (PDM_SPIN_US=0)
set -u
o=gpurun_out/r05f; mkdir -p $o
for r in 1 2; do
for sp in 0 200; do
PDM_SPIN_US=$sp timeout 300 python tools/exp/update_latency_probe.py > $o/lat_$sp.$r.json 2>>$o/err.txt; echo "lat $sp rc=$?" >> $o/status.txt
PDM_SPIN_US=$sp timeout 300 python tools/exp/small_update_probe.py > $o/small_$sp.$r.json 2>>$o/err.txt; echo "small $sp rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
