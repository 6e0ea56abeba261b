#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck (+ synccheck) over the small -m gpu
# cases: merges (raw, packed, flags/PDL, sparse D' to host), DT tile layouts,
# slab fold, pack, render.
set -u
o=gpurun_out/san; mkdir -p $o
CS=/usr/local/cuda/bin/compute-sanitizer
sel="test_distance_transform_golden or test_distance_transform_tile_layouts or test_worked_example or test_combine_empty_singleton_full or test_dprime_to_host_formats_and_pieces or test_packed_abi_many_planes or test_merge_packed_to_host_formats_and_pieces or test_merge_writes_stay_inside_the_map or test_merge_fused_zero_count or test_packed_merge_matches_oracle or test_combine_more_than_one_param_batch or test_volume_range_kernel or test_build_pdm_set"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
     python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$sel" -p no:cacheprovider \
     > $o/$tool.txt 2>&1; echo "$tool rc=$?" >> $o/status.txt
done
timeout 900 $CS --tool memcheck --target-processes all --print-limit 50 --error-exitcode 99 \
   python -m pytest tests/test_sharded.py tests/test_render.py -m gpu -q -x -p no:cacheprovider \
   > $o/memcheck_sharded_render.txt 2>&1; echo "memcheck_sharded_render rc=$?" >> $o/status.txt
