#!/usr/bin/env bash
set -u
o=gpurun_out/r02o; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed or merge or combine" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_main$r.jsonl 2> $o/bench_main.err; echo "bench main rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_pred.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_pred$r.jsonl 2> $o/bench_pred.err; echo "bench pred rc=$?" >> $o/status.txt
PDM_TILE_SKIP=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_noskip$r.jsonl 2> $o/bench_noskip.err; echo "bench noskip rc=$?" >> $o/status.txt
done
