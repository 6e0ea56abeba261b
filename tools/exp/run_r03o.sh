#!/usr/bin/env bash
set -u
o=gpurun_out/r03o; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
for kk in 4 0 2 6 8; do
PDM_RAW_MAX_K=$kk timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_k${kk}_$r.jsonl 2> $o/err.txt; echo "k$kk rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
