#!/usr/bin/env bash
set -u
o=gpurun_out/r04e; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench$r.jsonl 2> $o/err.txt; echo "bench rc=$?" >> $o/status.txt
done
cat $o/status.txt
