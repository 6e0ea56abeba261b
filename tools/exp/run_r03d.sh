#!/usr/bin/env bash
# A/B: pipelined merge (cp.async ring across tiles) vs the batch loop
set -u
o=gpurun_out/r03d; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or smoke or session" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_pipe$r.jsonl 2> $o/bench_pipe.err; echo "pipe rc=$?" >> $o/status.txt
PDM_MERGE_PIPE=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_old$r.jsonl 2> $o/bench_old.err; echo "old rc=$?" >> $o/status.txt
done
cat $o/status.txt
