#!/usr/bin/env bash
# sanity after container re-creation: GPU tests, smoke, bench, precompute
set -u
o=gpurun_out/r03a; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -x > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?" >> $o/status.txt
timeout 600 python bench.py > $o/bench_default.jsonl 2> $o/bench_default.err; echo "bench rc=$?" >> $o/status.txt
timeout 600 python tools/precompute_bench.py > $o/precompute.json 2>&1; echo "pre rc=$?" >> $o/status.txt
cat $o/status.txt
