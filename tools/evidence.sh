#!/usr/bin/env bash
# One GPU call that regenerates the round's measured evidence into gpurun_out/
# (copied into profiles/ afterwards).  Every ncu command runs only after the
# same program exited 0 without ncu in this call.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/evidence.sh r01'
set -u
tag=${1:-r01}
o=gpurun_out/$tag
mkdir -p "$o"
python -m pytest tests -m gpu -q > "$o/pytest_gpu.txt" 2>&1; echo "pytest rc=$?" >> "$o/status.txt"
python -c "import __graft_entry__ as g; g.smoke()" > "$o/smoke.txt" 2>&1; echo "smoke rc=$?" >> "$o/status.txt"
python bench.py > "$o/bench_default.jsonl" 2> "$o/bench_default.err"; echo "bench rc=$?" >> "$o/status.txt"
python bench.py --impl reference > "$o/bench_reference.jsonl" 2> "$o/bench_reference.err"; echo "ref rc=$?" >> "$o/status.txt"
python tools/precompute_bench.py > "$o/precompute.json" 2>&1; echo "pre rc=$?" >> "$o/status.txt"
python tools/merge_microbench.py --packed > "$o/merge_microbench.json" 2>&1; echo "mb rc=$?" >> "$o/status.txt"
python tools/configs_bench.py --cpu > "$o/configs.jsonl" 2>&1; echo "cfg rc=$?" >> "$o/status.txt"
python tools/recompute_probe.py > "$o/recompute_probe.json" 2>&1; echo "recompute rc=$?" >> "$o/status.txt"
python tools/host_path_probe.py > "$o/host_path_probe.json" 2>&1; echo "host path rc=$?" >> "$o/status.txt"
python tools/render_bench.py --reps 5 > "$o/render_bench.json" 2>&1; echo "render rc=$?" >> "$o/status.txt"
# launch list of the fused recompute (standard_distance_map, both modes)
python tools/exp/recompute_once.py && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file "$o/recompute_launches.csv" python tools/exp/recompute_once.py \
      > "$o/ncu_recompute.log" 2>&1; echo "ncu recompute rc=$?" >> "$o/status.txt"
# launch list of a short bench run (cold-cache, serialised)
python bench.py --steps 32 --warmup 3 --no-cpu-baseline > "$o/bench_short.jsonl" 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file "$o/bench_launches.csv" python bench.py --steps 32 --warmup 3 --no-cpu-baseline \
      > "$o/ncu_launches.log" 2>&1; echo "ncu launches rc=$?" >> "$o/status.txt"
# full capture of the k=32 packed merge inside the bench
ncu --set full --clock-control none --import-source on -k regex:combine_packed_flags -s 31 -c 1 \
    -o "$o/merge_k32_full" python bench.py --steps 32 --warmup 3 --no-cpu-baseline \
    > "$o/ncu_merge.log" 2>&1; echo "ncu merge rc=$?" >> "$o/status.txt"
# full capture of the precompute kernels (DT sweeps, apron)
python tools/precompute_bench.py --reps 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --kernel-name-base demangled \
      -k "regex:dt_tile_kernel|dt_dist1d_wide|apron_fast|pack_kernel|dt_expand" -c 8 \
      -o "$o/precompute_full" python tools/precompute_bench.py --reps 1 \
      > "$o/ncu_pre.log" 2>&1; echo "ncu pre rc=$?" >> "$o/status.txt"
# full capture of the voxel block scan (fused recompute's volume pass)
ncu --set full --clock-control none --import-source on -k regex:block_lut_fast -c 1 \
    -o "$o/blocklut_full" python tools/exp/recompute_once.py \
    > "$o/ncu_blocklut.log" 2>&1; echo "ncu blocklut rc=$?" >> "$o/status.txt"
cat "$o/status.txt"
