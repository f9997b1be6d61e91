set -u
mkdir -p gpurun_out
for W in 2 4 8; do
timeout 600 python bench.py --emulate-world $W --no-e2e --no-cpu --layers-json gpurun_out/layers_emu$W.json > gpurun_out/bench_emu$W.json 2>gpurun_out/bench_emu$W.err; echo "W=$W rc=$?"; tail -1 gpurun_out/bench_emu$W.json | head -c 400; echo
done
