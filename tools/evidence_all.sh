#!/bin/bash
# Full evidence pass (run under gpurun from the repo root): GPU tests, the full
# bench line (e2e, cpu_baseline, clocks), the reference arm, the emulated
# per-rank shards of the 2/4/8-GPU runs, the ncu launch list of one step, and
# `ncu --set full` of the top kernels (one launch each).  Each ncu run starts
# only after its command has exited 0 without ncu.
set -u
TAG=${1:-r1s}
LAYERS=${2:-stem,s2b0_3x3,s4b1_3x3,s4b1_1x1b,s4b1_1x1a,s3b1_3x3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests_rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py --layers-json gpurun_out/layers_$TAG.json > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo "bench_rc=$?"; tail -1 gpurun_out/bench_full_$TAG.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref_rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.json
for W in 2 4 8; do
  timeout 600 python bench.py --emulate-world $W --no-e2e --no-cpu --layers-json gpurun_out/layers_${TAG}_emu$W.json > gpurun_out/bench_${TAG}_emu$W.json 2>&1; echo "emu$W rc=$?"
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph --no-traffic"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"conv_" -s 53 -c 53 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu_launch_rc=$?"
timeout 300 python tools/run_layer.py --layer $LAYERS --once > gpurun_out/plain_full.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"conv_" -c 6 \
    -o gpurun_out/full_$TAG python tools/run_layer.py --layer $LAYERS --once > gpurun_out/ncu_full.log 2>&1
echo "ncu_full_rc=$?"
