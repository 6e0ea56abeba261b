#!/usr/bin/env bash
# A/B: tiles of a lap dealt round-robin over CTAs (SM balance) vs contiguous per CTA
set -u
o=gpurun_out/r04p; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2 3; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2> $o/err.txt; echo "base rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_pool.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_pool$r.jsonl 2>> $o/err.txt; echo "pool rc=$?" >> $o/status.txt
done
cat $o/status.txt
