#!/usr/bin/env bash
# A/B: 36 / 40 warps per SM (2 CTAs of 576 / 640 threads) vs 32 (1 CTA of 1024)
set -u
o=gpurun_out/r05a; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2> $o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in w36b5 w36b4 w40b4; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_$v$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
