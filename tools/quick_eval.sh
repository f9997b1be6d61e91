set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-e2e --no-cpu --layers-json gpurun_out/layers_s.json > gpurun_out/bench_s.json 2>gpurun_out/bench_s.err; echo "bench_rc=$?"; tail -1 gpurun_out/bench_s.json | head -c 300; echo
timeout 600 python bench.py --no-e2e --no-cpu --emulate-world 8 --layers-json gpurun_out/layers_s8.json > gpurun_out/bench_s8.json 2>&1; tail -1 gpurun_out/bench_s8.json | head -c 300; echo
timeout 300 python tools/run_layer.py --layer stem --once > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv_" -c 1 -o gpurun_out/full_stem python tools/run_layer.py --layer stem --once > gpurun_out/ncu_stem.log 2>&1; echo "ncu_rc=$?"
