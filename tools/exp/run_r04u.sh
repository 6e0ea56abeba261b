#!/usr/bin/env bash
# A/B: planes per batch 6 (default) / 7 / 8 at 1024 threads, 32-bit indices
set -u
o=gpurun_out/r04u; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or session or host or e2e or flags" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_b6_$r.jsonl 2> $o/err.txt; echo "b6 rc=$?" >> $o/status.txt
for v in b7 b8; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_${v}_$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
