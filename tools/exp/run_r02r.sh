#!/usr/bin/env bash
set -u
o=gpurun_out/r02r; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_main$r.jsonl 2> $o/bench_main.err; echo "bench main rc=$?" >> $o/status.txt
for v in v0 ahead2; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_$v$r.jsonl 2> $o/bench_$v.err; echo "bench $v rc=$?" >> $o/status.txt
done
PDM_TILE_SKIP=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_noskip$r.jsonl 2> $o/bench_noskip.err; echo "bench noskip rc=$?" >> $o/status.txt
done
