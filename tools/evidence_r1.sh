#!/bin/bash
# Round-1 evidence pass, part 1 (run under gpurun from the repo root; ONE ncu run):
# GPU tests, the full bench line, the reference arm, and the ncu launch list of one step.
set -u
TAG=${1:-r1m}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --layers-json gpurun_out/layers_$TAG.json > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo "bench_rc=$?"; tail -1 gpurun_out/bench_full_$TAG.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref_rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.json
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"conv_" -s 53 -c 53 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu_launch_rc=$?"
