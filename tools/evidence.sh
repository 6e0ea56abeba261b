#!/usr/bin/env bash
# One GPU call that regenerates the round's measured evidence into gpurun_out/
# (copied into profiles/ afterwards).  Every ncu command runs only after the
# same program exited 0 without ncu in this call.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/evidence.sh r02'
set -u
tag=${1:-r02}
o=gpurun_out/$tag
mkdir -p "$o"
python -m pytest tests -m gpu -q > "$o/pytest_gpu.txt" 2>&1; echo "pytest rc=$?" >> "$o/status.txt"
python -c "import __graft_entry__ as g; g.smoke()" > "$o/smoke.txt" 2>&1; echo "smoke rc=$?" >> "$o/status.txt"
python bench.py > "$o/bench_default.jsonl" 2> "$o/bench_default.err"; echo "bench rc=$?" >> "$o/status.txt"
python bench.py --impl reference > "$o/bench_reference.jsonl" 2> "$o/bench_reference.err"; echo "ref rc=$?" >> "$o/status.txt"
python bench.py --steps 20 --warmup 5 > "$o/bench_driver_shape.jsonl" 2> "$o/bench_driver_shape.err"; echo "bench20 rc=$?" >> "$o/status.txt"
python bench.py --steps 32 --warmup 5 --config d --no-cpu-baseline > "$o/bench_config_d.jsonl" 2> "$o/bench_config_d.err"; echo "bench d rc=$?" >> "$o/status.txt"
python tools/precompute_bench.py > "$o/precompute.json" 2>&1; echo "pre rc=$?" >> "$o/status.txt"
python tools/configs_bench.py --cpu > "$o/configs.jsonl" 2>&1; echo "cfg rc=$?" >> "$o/status.txt"
python tools/recompute_probe.py > "$o/recompute_probe.json" 2>&1; echo "recompute rc=$?" >> "$o/status.txt"
python tools/exp/e2e_probe.py > "$o/e2e_probe.json" 2>&1; echo "e2e probe rc=$?" >> "$o/status.txt"
python tools/exp/small_update_probe.py > "$o/small_update.json" 2>&1; echo "small rc=$?" >> "$o/status.txt"
PDM_REF_SUITE_REPORT=$o/ref_suite.json python -m pytest tests/test_reference_suite.py -q -s > "$o/ref_suite.txt" 2>&1; echo "refsuite rc=$?" >> "$o/status.txt"
bash tools/ref_cli_bench.sh "$o/refcli" > "$o/ref_cli.txt" 2>&1; echo "refcli rc=$?" >> "$o/status.txt"
# per-k DRAM traffic of the merge over the bench's 32-step TF sequence
ks=$(seq -s ' ' 1 32)
python tools/exp/merge_once.py $ks > "$o/merge_seq_plain.log" 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:combine_packed_flags --csv --log-file "$o/merge_seq.csv" python tools/exp/merge_once.py $ks \
      > "$o/ncu_merge_seq.log" 2>&1; echo "ncu merge seq rc=$?" >> "$o/status.txt"
# full captures of the merge at k = 8, 16, 32 (same TFs as the bench's steps)
python tools/exp/merge_once.py 8 16 32 > "$o/merge3_plain.log" 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:combine_packed_flags -c 3 \
      -o "$o/merge_k8_16_32_full" python tools/exp/merge_once.py 8 16 32 \
      > "$o/ncu_merge_full.log" 2>&1; echo "ncu merge full rc=$?" >> "$o/status.txt"
# full capture of the precompute kernels (apron POM, expand, DT passes)
python tools/exp/precompute_once.py 1 > "$o/pre_plain.log" 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k "regex:apron_fast|dt_tmem|dt_x_mask|dt_tile|tile_bounds" -c 6 \
      -o "$o/precompute_full" python tools/exp/precompute_once.py 1 \
      > "$o/ncu_pre.log" 2>&1; echo "ncu pre rc=$?" >> "$o/status.txt"
# launch list of a short bench run (cold-cache, serialised)
python bench.py --steps 32 --warmup 3 --no-cpu-baseline > "$o/bench_short.jsonl" 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file "$o/bench_launches.csv" python bench.py --steps 32 --warmup 3 --no-cpu-baseline \
      > "$o/ncu_launches.log" 2>&1; echo "ncu launches rc=$?" >> "$o/status.txt"
cat "$o/status.txt"
