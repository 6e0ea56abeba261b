#!/usr/bin/env bash
set -u
o=gpurun_out/r02m; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
V=paper_2407_21552_b200/lib/variants
for v in static static_all claim8 claim4; do
  PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_$v.jsonl 2> $o/bench_$v.err; echo "bench $v rc=$?" >> $o/status.txt
done
for v in static claim8; do
  PDM_TILE_SKIP=0 PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_${v}_noskip.jsonl 2> $o/bench_${v}_noskip.err; echo "bench $v noskip rc=$?" >> $o/status.txt
done
