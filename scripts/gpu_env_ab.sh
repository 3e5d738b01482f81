#!/usr/bin/env bash
# GPU tests, then a same-box A/B of an env switch on the bench.
# Usage: gpurun -- bash scripts/gpu_env_ab.sh <tag> <VAR> "<v1> <v2>" [pytest -k expr | -]
set -u
TAG=${1:-eab}; VAR=${2:-ROTOR_GRAPH}; VALS=${3:-"1 0"}; K=${4:-}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { tail -20 "$OUT/build.log"; exit 1; }
if [ "$K" != "-" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu.log)"; grep -E "^FAILED|Error" "$OUT/pytest_gpu.log" | head -5
fi
for rep in 1 2; do for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > $OUT/bench_${v}_$rep.json 2> $OUT/bench_${v}_$rep.err
  echo "$VAR=$v $(grep -o '"ms_per_step": [0-9.]*' $OUT/bench_${v}_$rep.json | head -2 | tr '\n' ' ') $(grep -o '"middle_ms_per_step": [0-9.]*' $OUT/bench_${v}_$rep.json)"
done; done
