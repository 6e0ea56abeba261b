#!/usr/bin/env bash
set -u
o=gpurun_out/r03n; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or session or smoke or e2e or host" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2 3; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_dyn$r.jsonl 2> $o/err.txt; echo "dyn rc=$?" >> $o/status.txt
PDM_MERGE_DYNAMIC=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_static$r.jsonl 2>> $o/err.txt; echo "static rc=$?" >> $o/status.txt
done
cat $o/status.txt
