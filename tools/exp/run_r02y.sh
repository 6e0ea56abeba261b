#!/usr/bin/env bash
set -u
o=gpurun_out/r02y; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_host_api.py tests/test_session.py -m gpu -q -x > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
python tools/exp/small_update_probe.py > $o/small_update.json 2>&1; echo "small rc=$?" >> $o/status.txt
python tools/exp/small_update_probe.py --breakdown > $o/small_bd.txt 2>&1; echo "bd rc=$?" >> $o/status.txt
PDM_REF_SUITE_REPORT=$o/ref_suite.json timeout 1200 python -m pytest tests/test_reference_suite.py -q -s > $o/ref_suite.txt 2>&1; echo "refsuite rc=$?" >> $o/status.txt
V=paper_2407_21552_b200/lib/variants
for v in novote b4c4 b8c3; do
PDM_LIB_PATH=$V/libpdm_b200_$v.so timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_$v.jsonl 2> $o/bench_$v.err; echo "bench $v rc=$?" >> $o/status.txt
done
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline --no-parity > $o/bench_main.jsonl 2> $o/bench_main.err; echo "bench main rc=$?" >> $o/status.txt
