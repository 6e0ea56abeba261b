#!/usr/bin/env bash
set -u
o=gpurun_out/r02n; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed or merge or combine" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
V=paper_2407_21552_b200/lib/variants
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_main.jsonl 2> $o/bench_main.err; echo "bench main rc=$?" >> $o/status.txt
PDM_TILE_SKIP=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_noskip.jsonl 2> $o/bench_noskip.err; echo "bench noskip rc=$?" >> $o/status.txt
for v in all nofetch; do
  PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_$v.jsonl 2> $o/bench_$v.err; echo "bench $v rc=$?" >> $o/status.txt
done
