#!/usr/bin/env bash
set -u
o=gpurun_out/r04j; mkdir -p $o
timeout 900 python -m pytest tests/test_render.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 900 python tools/render_bench.py --reps 5 > $o/render.json 2>&1; echo "render rc=$?" >> $o/status.txt
cat $o/status.txt
