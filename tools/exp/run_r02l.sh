#!/usr/bin/env bash
set -u
o=gpurun_out/r02l; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
PDM_TILE_SKIP=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_noskip.jsonl 2> $o/bench_noskip.err; echo "bench noskip rc=$?" >> $o/status.txt
