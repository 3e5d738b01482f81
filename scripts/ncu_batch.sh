#!/usr/bin/env bash
# One ncu --set full capture of k_batch (config 5) from the working tree.
# Usage: gpurun -- bash scripts/ncu_batch.sh <tag>
set -u
TAG=${1:-nb}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o $OUT/k_batch \
  python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1; echo ncu rc=$?
