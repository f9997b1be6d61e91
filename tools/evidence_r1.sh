#!/bin/bash
# Round-1 evidence pass (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref_rc=$?"; tail -1 gpurun_out/bench_ref.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv_" -s 53 -c 53 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
for L in stem s2b0_3x3 s4b1_3x3 s2b0_1x1b; do
  timeout 300 python tools/run_layer.py --layer $L --reps 2 > gpurun_out/plain_$L.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_" -s 1 -c 1 \
      -o gpurun_out/full_$L python tools/run_layer.py --layer $L --reps 2 > gpurun_out/ncu_full_$L.log 2>&1
  echo "ncu_full_${L}_rc=$?"
done
