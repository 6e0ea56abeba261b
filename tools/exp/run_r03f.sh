#!/usr/bin/env bash
# A/B: double-buffered compacted merge (B=4, 3 CTAs) vs batch loop; variants
set -u
o=gpurun_out/r03f; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "merge or packed or combine or smoke or session" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_db$r.jsonl 2> $o/err_db.txt; echo "db rc=$?" >> $o/status.txt
PDM_MERGE_DB=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_old$r.jsonl 2> $o/err_old.txt; echo "old rc=$?" >> $o/status.txt
for v in b6c2 b2c4 b3c3; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_$v$r.jsonl 2> $o/err_$v.txt; echo "$v rc=$?" >> $o/status.txt
done
done
cat $o/status.txt
