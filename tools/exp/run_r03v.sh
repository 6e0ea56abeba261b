#!/usr/bin/env bash
# apron kernel with TMA plane loads: parity + A/B + ncu
set -u
o=gpurun_out/r03v; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "apron or min_max or range or occupancy or build_pdm_set or precompute_kernels or standard or config or sharded" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_tma_$r.json 2>&1; echo "pre rc=$?" >> $o/status.txt
PDM_APRON_TMA=0 timeout 300 python tools/precompute_bench.py > $o/pre_cpa_$r.json 2>&1; echo "pre cpa rc=$?" >> $o/status.txt
done
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:apron_fast" -c 1 \
    -o $o/apron python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
