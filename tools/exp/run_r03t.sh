#!/usr/bin/env bash
# x pass from the mask with TMEM-parked forward runs: parity + A/B
set -u
o=gpurun_out/r03t; mkdir -p $o
V=paper_2407_21552_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "build_pdm_set or precompute or distance or config or golden or tile_bounds or sharded or slab" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
for r in 1 2; do
timeout 300 python tools/precompute_bench.py > $o/pre_tmem_$r.json 2>&1; echo "pre rc=$?" >> $o/status.txt
PDM_LIB_PATH=$V/libpdm_b200_c3.so timeout 300 python tools/precompute_bench.py > $o/pre_c3_$r.json 2>&1; echo "c3 rc=$?" >> $o/status.txt
PDM_DT_XMASK_TMEM=0 timeout 300 python tools/precompute_bench.py > $o/pre_smem_$r.json 2>&1; echo "smem rc=$?" >> $o/status.txt
done
python tools/exp/precompute_once.py 1 > $o/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dt_x_mask" -c 1 \
    -o $o/xmt python tools/exp/precompute_once.py 1 > $o/ncu_p.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
cat $o/status.txt
