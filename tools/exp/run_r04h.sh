#!/usr/bin/env bash
# A/B: per-warp bulk-copy ring merge (PDM_MERGE_BULK=1) vs the batch loop
set -u
o=gpurun_out/r04h; mkdir -p $o
PDM_MERGE_BULK=1 timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or flags" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2> $o/err.txt; echo "base rc=$?" >> $o/status.txt
PDM_MERGE_BULK=1 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_bulk$r.jsonl 2>> $o/err.txt; echo "bulk rc=$?" >> $o/status.txt
done
cat $o/status.txt
