#!/usr/bin/env bash
set -u
o=gpurun_out/r02d; mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_reference_suite.py > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
PDM_REF_SUITE_REPORT=$o/ref_suite.json timeout 1200 python -m pytest tests/test_reference_suite.py -q -s > $o/ref_suite.txt 2>&1; echo "refsuite rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 32 --warmup 5 --config d --no-cpu-baseline > $o/bench_d.jsonl 2> $o/bench_d.err; echo "bench d rc=$?" >> $o/status.txt
