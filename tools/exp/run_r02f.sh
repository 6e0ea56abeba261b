#!/usr/bin/env bash
set -u
o=gpurun_out/r02f; mkdir -p $o
python tools/exp/small_update_probe.py > $o/small_update.json 2>&1; echo "small rc=$?" >> $o/status.txt
python tools/exp/select_probe.py > $o/select_probe.json 2>&1; echo "sel rc=$?" >> $o/status.txt
python tools/exp/e2e_probe.py > $o/e2e_probe.json 2>&1; echo "probe rc=$?" >> $o/status.txt
