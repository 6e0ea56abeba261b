#!/usr/bin/env bash
# A/B: raw small-k path out of line (packed loop spill-free) vs inlined (HEAD)
set -u
o=gpurun_out/r04v; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or flags" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2 3; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_new$r.jsonl 2> $o/err.txt; echo "new rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_head.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_head$r.jsonl 2>> $o/err.txt; echo "head rc=$?" >> $o/status.txt
done
cat $o/status.txt
