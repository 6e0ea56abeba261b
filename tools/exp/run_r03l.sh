#!/usr/bin/env bash
set -u
o=gpurun_out/r03l; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
PDM_LIB_PATH=$V/libpdm_b200_viadd.so timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2 3; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_base$r.jsonl 2> $o/err.txt; echo "base rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_viadd.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_viadd$r.jsonl 2>> $o/err.txt; echo "viadd rc=$?" >> $o/status.txt
done
cat $o/status.txt
