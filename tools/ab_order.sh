# same-box A/B of the sweep's launch order / jobs / grid snapping (bench.py diagnostics)
run() { echo "$*: $(timeout 300 python bench.py --no-e2e --no-cpu --no-traffic --no-parity "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["run"].get("sweep_ctas_per_launch"))')"; }
for rep in 1 2; do
for O in sweep mix; do
  for J in 0 2; do
    run --launch-order $O --sweep-jobs $J --no-snap
    run --launch-order $O --sweep-jobs $J
  done
done
done
for W in 2 8; do
for O in sweep mix; do
  run --emulate-world $W --launch-order $O --no-snap
  run --emulate-world $W --launch-order $O
done
done
