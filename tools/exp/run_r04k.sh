#!/usr/bin/env bash
# host alpha gather: pool unit size A/B through the e2e bench
set -u
o=gpurun_out/r04k; mkdir -p $o
for r in 1 2; do
for u in 4096 1024 512; do
PDM_GATHER_UNIT=$u timeout 600 python bench.py --steps 64 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_u${u}_$r.jsonl 2> $o/err.txt; echo "u$u rc=$?" >> $o/status.txt
done; done
nproc > $o/nproc.txt
cat $o/status.txt
