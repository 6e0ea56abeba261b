#!/usr/bin/env bash
# timing probes (wrong results by construction): which stream bounds the merge
set -u
o=gpurun_out/r03m; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2> $o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in bl2 nl2; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_$v$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
