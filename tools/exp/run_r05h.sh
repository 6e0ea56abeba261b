#!/usr/bin/env bash
# A/B: packed merge at 28 warps per SM (one CTA of 896 threads, 72 registers)
# with 6 / 7 / 8 planes per batch vs 32 warps (1024 threads, 64 registers, 6)
set -u
o=gpurun_out/r05h; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2>> $o/err.txt; echo "base rc=$?" >> $o/status.txt
for v in p28b6 p28b7 p28b8; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_$v$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
