#!/usr/bin/env bash
set -u
o=gpurun_out/r02x; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_size.py tests/test_gpu_properties.py tests/test_sharded.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
python tools/precompute_bench.py > $o/pre_main.json 2>&1; echo "pre rc=$?" >> $o/status.txt
