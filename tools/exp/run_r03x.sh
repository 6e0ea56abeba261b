#!/usr/bin/env bash
set -u
o=gpurun_out/r03x; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?" >> $o/status.txt
timeout 600 python bench.py > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
cat $o/status.txt
