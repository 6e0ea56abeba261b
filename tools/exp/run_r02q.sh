#!/usr/bin/env bash
set -u
o=gpurun_out/r02q; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py tests/test_session.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench_main$r.jsonl 2> $o/bench_main.err; echo "bench main rc=$?" >> $o/status.txt
PDM_TILE_SKIP=0 timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_noskip$r.jsonl 2> $o/bench_noskip.err; echo "bench noskip rc=$?" >> $o/status.txt
done
