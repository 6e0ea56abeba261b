#!/usr/bin/env bash
set -u
o=gpurun_out/r02e; mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_reference_suite.py > $o/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $o/status.txt
PDM_REF_SUITE_REPORT=$o/ref_suite.json timeout 1200 python -m pytest tests/test_reference_suite.py -q -s > $o/ref_suite.txt 2>&1; echo "refsuite rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
timeout 600 python bench.py --steps 32 --warmup 5 --config d --no-cpu-baseline > $o/bench_d.jsonl 2> $o/bench_d.err; echo "bench d rc=$?" >> $o/status.txt
timeout 900 bash tools/ref_cli_bench.sh $o/refcli > $o/ref_cli.txt 2>&1; echo "refcli rc=$?" >> $o/status.txt
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_ref.jsonl 2> $o/bench_ref.err; echo "benchref rc=$?" >> $o/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/ncu.log 2>&1; echo "ncu rc=$?" >> $o/status.txt
