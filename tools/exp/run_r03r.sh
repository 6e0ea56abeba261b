#!/usr/bin/env bash
# A/B: chunked tile claims (1/2/4 tiles per claim, first chunk static) vs static split
set -u
o=gpurun_out/r03r; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
PDM_LIB_PATH=$V/libpdm_b200_dyn2.so timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or session" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_static$r.jsonl 2> $o/err.txt; echo "static rc=$?" >> $o/status.txt
for v in dyn1 dyn2 dyn4; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_$v$r.jsonl 2>> $o/err.txt; echo "$v rc=$?" >> $o/status.txt
done; done
cat $o/status.txt
