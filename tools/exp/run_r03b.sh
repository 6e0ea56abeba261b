#!/usr/bin/env bash
set -u
o=gpurun_out/r03b; mkdir -p $o
timeout 300 python tools/exp/small_update_probe.py > $o/small.json 2>&1; echo "small rc=$?" >> $o/status.txt
timeout 300 python tools/exp/small_update_probe.py --breakdown > $o/breakdown.txt 2>&1; echo "bd rc=$?" >> $o/status.txt
cat $o/status.txt
