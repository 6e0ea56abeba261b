#!/usr/bin/env bash
set -u
o=gpurun_out/r02h; mkdir -p $o
python tools/exp/small_update_probe.py --breakdown > $o/small_breakdown.txt 2>&1; echo "bd rc=$?" >> $o/status.txt
python tools/exp/e2e_probe.py > $o/e2e_probe.json 2>&1; echo "probe rc=$?" >> $o/status.txt
python tools/exp/select_probe.py > $o/select_probe.json 2>&1; echo "sel rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
