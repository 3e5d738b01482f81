#!/usr/bin/env bash
# Same-box A/B of the working tree ("new") against abtest/ (a build of HEAD, "old").
# Usage: gpurun -- bash scripts/ab.sh <tag> [pytest -k expr]
set -u
TAG=${1:-ab}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
if [ -n "${2:-}" ]; then
  timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "$2" > "$OUT/p1.log" 2>&1; tail -1 "$OUT/p1.log"
fi
for v in new old new old; do
  if [ $v = old ]; then (cd abtest && timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > ../$OUT/bench_$v.json 2>&1)
  else timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > $OUT/bench_$v.json 2>&1; fi
  echo $v $(grep -o '"ms_per_step": [0-9.]*' $OUT/bench_$v.json | head -1) $(grep -o '"middle_ms_per_step": [0-9.]*' $OUT/bench_$v.json)
done
