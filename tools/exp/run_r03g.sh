#!/usr/bin/env bash
# TMEM DT sweeps: parity + precompute A/B
set -u
o=gpurun_out/r03g; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "distance_transform or precompute_kernels or build_pdm_set or tile_bounds or standard" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 300 python tools/precompute_bench.py > $o/pre_tmem.json 2>&1; echo "pre rc=$?" >> $o/status.txt
PDM_DT_TMEM=0 timeout 300 python tools/precompute_bench.py > $o/pre_old.json 2>&1; echo "pre old rc=$?" >> $o/status.txt
timeout 300 python tools/precompute_bench.py > $o/pre_tmem2.json 2>&1; echo "pre rc=$?" >> $o/status.txt
cat $o/status.txt
