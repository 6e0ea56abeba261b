#!/usr/bin/env bash
# A/B: 32 warps per SM (1024-thread CTA, 64 registers, spills) vs 24
set -u
o=gpurun_out/r04t; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2> $o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in w32b4 w40b4 w32b5; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_$v$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
