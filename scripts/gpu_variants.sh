#!/usr/bin/env bash
# A/B timing of kernel variants selected by environment variables (run on the GPU box).
# Usage: VAR=ROTOR_LEAF VALUES="row tab tabr" PYTEST_K=tiled bash scripts/gpu_variants.sh <tag>
set -u
TAG=${1:-v}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
for V in ${VALUES}; do
  if [ -n "${PYTEST_K:-}" ]; then
    env $VAR=$V timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > "$OUT/pytest_$V.log" 2>&1
    echo "$VAR=$V pytest rc=$? $(tail -1 "$OUT/pytest_$V.log")"
  fi
  env $VAR=$V ROTOR_KERNEL=${KERNEL:-tiled} timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > "$OUT/bench_$V.json" 2> "$OUT/bench_$V.err"
  python - "$OUT/bench_$V.json" "$VAR=$V" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "ms_per_step %.2f fill_ms %.2f frac %.3f" % (d["ms_per_step"], d["fill_ms"], d["roofline"]["frac"]))
except Exception as e:
    print(sys.argv[2], "bench failed", e)
PY
done
