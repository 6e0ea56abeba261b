#!/usr/bin/env bash
set -u
o=gpurun_out/r04c; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "distance_transform or precompute_kernels or build_pdm_set or tile_bounds or random_volumes or config" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 600 python tools/precompute_bench.py --dims 2048 2048 2048 --reps 2 > $o/pre_d.json 2>&1; echo "pre d rc=$?" >> $o/status.txt
PDM_DT_XMASK=0 timeout 600 python tools/precompute_bench.py --dims 2048 2048 2048 --reps 2 > $o/pre_d_old.json 2>&1; echo "pre d old rc=$?" >> $o/status.txt
timeout 300 python tools/precompute_bench.py > $o/pre_c.json 2>&1; echo "pre c rc=$?" >> $o/status.txt
cat $o/status.txt
