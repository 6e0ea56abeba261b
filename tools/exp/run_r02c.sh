#!/usr/bin/env bash
set -u
o=gpurun_out/r02c; mkdir -p $o
python tools/exp/select_probe.py > $o/select_probe.json 2>&1; echo "sel rc=$?" >> $o/status.txt
python tools/exp/e2e_probe.py > $o/e2e_probe.json 2>&1; echo "probe rc=$?" >> $o/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_persistence_interop.py tests/test_session.py -m gpu -q -x > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
PDM_REF_SUITE_REPORT=$o/ref_suite.json timeout 1200 python -m pytest tests/test_reference_suite.py -q -s > $o/ref_suite.txt 2>&1; echo "refsuite rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
