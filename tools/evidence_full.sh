#!/bin/bash
# Evidence pass, part 2 (ONE ncu run): `ncu --set full` of the top kernels of the step, one launch each.
set -u
TAG=${1:-r1m}
LAYERS=${2:-stem,s2b0_3x3,s4b1_3x3,s4b1_1x1b,s3b1_3x3}
mkdir -p gpurun_out
timeout 300 python tools/run_layer.py --layer $LAYERS --once > gpurun_out/plain_full.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_" -c 5 \
    -o gpurun_out/full_$TAG python tools/run_layer.py --layer $LAYERS --once > gpurun_out/ncu_full.log 2>&1
echo "ncu_full_rc=$?"
