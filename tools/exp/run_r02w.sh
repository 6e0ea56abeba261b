#!/usr/bin/env bash
set -u
o=gpurun_out/r02w; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py tests/test_sharded.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
V=paper_2407_21552_b200/lib/variants
python tools/precompute_bench.py > $o/pre_main.json 2>&1; echo "pre rc=$?" >> $o/status.txt
for v in ring3 ring4; do PDM_LIB_PATH=$V/libpdm_b200_$v.so python tools/precompute_bench.py > $o/pre_$v.json 2>&1; echo "pre $v rc=$?" >> $o/status.txt; done
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
