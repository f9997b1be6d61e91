#!/bin/bash
# Build the microbenchmarks / probes in tools/ (sm_100a) and, with "run", record their output
# under profiles/r1/ (run on a GPU box: gpurun -- 'bash tools/build_bench.sh run').
set -eu
cd "$(dirname "$0")/.."
for t in mma_bench tma_bench l2_bench store_bench desc_probe m64_probe; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc \
       tools/$t.cu -o tools/$t -lcuda 2>/dev/null
done
if [ "${1:-}" = "run" ]; then
  mkdir -p gpurun_out
  for t in mma_bench tma_bench l2_bench store_bench desc_probe m64_probe; do
    timeout 120 ./tools/$t > gpurun_out/$t.txt 2>&1; echo "$t rc=$?"
  done
fi
