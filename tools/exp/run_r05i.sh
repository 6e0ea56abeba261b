#!/usr/bin/env bash
# A/B: packed merge at 24 / 26 / 28 warps per SM with 8 planes per batch vs 32 warps with 6
set -u
o=gpurun_out/r05i; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2>> $o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in p28b8 p24b8 p26b8; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_$v$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
