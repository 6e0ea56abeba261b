#!/usr/bin/env bash
set -u
o=gpurun_out/r04l; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
timeout 900 python -m pytest tests/test_render.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 900 python tools/render_bench.py --reps 5 --cpu-rows 1 > $o/render_m1_$r.json 2>&1; echo "m1 rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_m5.so timeout 900 python tools/render_bench.py --reps 5 --cpu-rows 1 > $o/render_m5_$r.json 2>&1; echo "m5 rc=$?" >> $o/status.txt
done
cat $o/status.txt
