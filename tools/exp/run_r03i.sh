#!/usr/bin/env bash
set -u
o=gpurun_out/r03i; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "distance_transform or precompute_kernels or build_pdm_set or tile_bounds or standard" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
timeout 300 python tools/precompute_bench.py > $o/pre_tmem.json 2>&1; echo "pre rc=$?" >> $o/status.txt
PDM_DT_TMEM=0 timeout 300 python tools/precompute_bench.py > $o/pre_old.json 2>&1; echo "pre old rc=$?" >> $o/status.txt
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dt_tmem" -c 2 \
    -o $o/tmem python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
