#!/bin/bash
# Build and run the merge-variant experiment (GPU box).  Usage:
#   bash tools/exp/run_merge_variants.sh [variant] [reps]
set -e
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/merge_variants merge_variants.cu
timeout 300 /tmp/merge_variants "$@"
