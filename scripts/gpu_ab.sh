#!/usr/bin/env bash
# GPU tests of the working tree, then a same-box A/B of its bench against
# abtest/ (a build of the baseline).  Usage: gpurun -- bash scripts/gpu_ab.sh <tag> [pytest -k expr]
set -u
TAG=${1:-ab}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { tail -20 "$OUT/build.log"; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${2:+-k "$2"} > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu.log)"; grep -E "FAILED|Error" "$OUT/pytest_gpu.log" | head -5
bash scripts/ab.sh "$TAG"
