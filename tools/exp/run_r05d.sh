#!/usr/bin/env bash
# TMEM sweep shape chosen by job size: parity with each shape forced, timings
set -u
o=gpurun_out/r05d; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $o/parity_auto.txt 2>&1; echo "parity auto rc=$?" >> $o/status.txt
PDM_DT_TMEM_BIG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $o/parity_big.txt 2>&1; echo "parity big rc=$?" >> $o/status.txt
PDM_DT_TMEM_BIG=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "pdm_set or build or config" > $o/parity_small.txt 2>&1; echo "parity small rc=$?" >> $o/status.txt
for r in 1 2; do timeout 300 python tools/precompute_bench.py > $o/pre$r.json 2>>$o/err.txt; echo "pre rc=$?" >> $o/status.txt; done
timeout 300 python tools/recompute_probe.py > $o/recompute.json 2>>$o/err.txt; echo "recompute rc=$?" >> $o/status.txt
timeout 600 python tools/precompute_bench.py --dims 2048 2048 2048 --reps 2 > $o/pre_d.json 2>>$o/err.txt; echo "d rc=$?" >> $o/status.txt
cat $o/status.txt
