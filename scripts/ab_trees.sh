#!/usr/bin/env bash
# Same-box comparison of prebuilt trees (each a copy of the repo with its own
# in-tree .so): bench each twice, interleaved.  Usage: gpurun -- bash scripts/ab_trees.sh <tag> <dir>...
set -u
TAG=$1; shift; OUT=$PWD/gpurun_out/$TAG; mkdir -p "$OUT"
for rep in 1 2; do for t in "$@"; do
  (cd "$t" && timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > "$OUT/bench_$(basename $t)_$rep.json" 2>&1)
  echo "$t $(grep -o '"ms_per_step": [0-9.]*' "$OUT/bench_$(basename $t)_$rep.json" | head -1)"
done; done
