#!/usr/bin/env bash
set -u
o=gpurun_out/r02i; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $o/pytest_parity.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
python tools/exp/small_update_probe.py > $o/small_update.json 2>&1; echo "small rc=$?" >> $o/status.txt
python tools/exp/small_update_probe.py --breakdown > $o/small_breakdown.txt 2>&1; echo "bd rc=$?" >> $o/status.txt
PDM_REF_SUITE_REPORT=$o/ref_suite.json timeout 1200 python -m pytest tests/test_reference_suite.py -q -s > $o/ref_suite.txt 2>&1; echo "refsuite rc=$?" >> $o/status.txt
