#!/usr/bin/env bash
set -u
o=gpurun_out/r02z; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
for r in 1 2; do
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_main$r.jsonl 2> $o/bench_main.err; echo "bench main rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_pf.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_pf$r.jsonl 2> $o/bench_pf.err; echo "bench pf rc=$?" >> $o/status.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "precompute_kernels_write or tile_bounds or packed_abi" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
