#!/usr/bin/env bash
set -u
o=gpurun_out/r04f; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "flags_merge or packed_merge or merge" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2 3; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench$r.jsonl 2> $o/err.txt; echo "bench rc=$?" >> $o/status.txt
done
cat $o/status.txt
