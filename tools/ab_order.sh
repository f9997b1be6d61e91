# same-box A/B of the sweep's launch order / jobs (bench.py diagnostics); usage: bash tools/ab_order.sh
run() { echo "$*: $(timeout 300 python bench.py --no-e2e --no-cpu --no-traffic --no-parity "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["run"].get("sweep_ctas_per_launch"))')"; }
for rep in 1 2; do
  for J in 1.5 1.75 2 2.33 2.67; do
    run --launch-order mix --sweep-jobs $J
  done
  run --launch-order sweep --sweep-jobs 2.67
done
for W in 2 4 8; do
  for J in 3 4 5; do
    run --emulate-world $W --launch-order mix --sweep-jobs $J
  done
done
