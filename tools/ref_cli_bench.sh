#!/usr/bin/env bash
# The reference's own `pdmrender bench` (the producer of the paper's update
# table, bench.py:192-249) run UNMODIFIED through the drop-in overlay on the
# GPU box: build_pdm_set / standard_distance_map / select_partitions / combine
# are this repo's CUDA path, every call returning completed device work, so
# the reference's own perf_counter timers (measure_ms) measure the GPU work.
#   tools/ref_cli_bench.sh OUT_DIR
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
REF="$ROOT/baseline/_ref/pdmrender"
[ -d "$REF" ] || REF=/root/reference/pkg/src/pdmrender
export PYTHONPATH="$ROOT/integration:$ROOT" PDMRENDER_REF="$REF" NUMBA_CACHE_DIR=/tmp/numba_cache
for occ in voxel range-apron; do
  python -m pdmrender.cli bench --synth sphere_shell --dims 512 --seed 0 --counts 16,32,64 \
      --tfs tf1,tf2,tf3,tf4 --occupancy "$occ" --repeats 20 --report json \
      --out "$OUT/pdmrender_bench_512_${occ}.json"
done
python -m pdmrender.cli bench --synth sphere_shell --dims 256 --seed 0 --counts 16,32,64,128,256 \
    --occupancy voxel --repeats 20 --report csv --out "$OUT/pdmrender_bench_256_voxel.csv"
echo "reports in $OUT"
