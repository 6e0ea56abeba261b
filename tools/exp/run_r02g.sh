#!/usr/bin/env bash
set -u
o=gpurun_out/r02g; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_view or dprime_to_host or merge_packed_to_host or eager or select" > $o/pytest_sel.txt 2>&1; echo "pytest_sel rc=$?" >> $o/status.txt
python tools/exp/small_update_probe.py > $o/small_update.json 2>&1; echo "small rc=$?" >> $o/status.txt
PDM_SELECT_DMA=1 python tools/exp/small_update_probe.py > $o/small_update_dma.json 2>&1; echo "small dma rc=$?" >> $o/status.txt
python tools/exp/select_probe.py > $o/select_probe.json 2>&1; echo "sel rc=$?" >> $o/status.txt
PDM_SELECT_DMA=1 python tools/exp/select_probe.py > $o/select_probe_dma.json 2>&1; echo "sel dma rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
PDM_HOST_SPECULATE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_nospec.jsonl 2> $o/bench_nospec.err; echo "bench nospec rc=$?" >> $o/status.txt
PDM_REF_SUITE_REPORT=$o/ref_suite.json timeout 1200 python -m pytest tests/test_reference_suite.py -q -s > $o/ref_suite.txt 2>&1; echo "refsuite rc=$?" >> $o/status.txt
