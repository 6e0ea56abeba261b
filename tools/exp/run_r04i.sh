#!/usr/bin/env bash
set -u
o=gpurun_out/r04i; mkdir -p $o
timeout 900 python tools/render_bench.py --reps 5 > $o/render.json 2>&1; echo "render rc=$?" >> $o/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_rays -c 1 -o $o/march python tools/render_bench.py --reps 1 --cpu-rows 1 > $o/ncu.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
