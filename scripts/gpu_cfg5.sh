#!/usr/bin/env bash
# Config-5 A/B: bench --config 5 over VALUES of VAR (batched sweep).
set -u
TAG=${1:-c5}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { tail -30 "$OUT/build.log"; exit 1; }
if [ -n "${PYTEST_K:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > "$OUT/pytest.log" 2>&1
  echo "pytest rc=$? $(tail -1 "$OUT/pytest.log")"
fi
for V in ${VALUES:-default}; do
  if [ "$V" = default ]; then E=""; else E="${VAR}=$V"; fi
  env $E timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > "$OUT/bench_$V.json" 2> "$OUT/bench_$V.err"
  echo "${E:-default} $(grep -o '"ms_per_step": [0-9.]*' $OUT/bench_$V.json) $(grep -o '"value": [0-9.e+]*' $OUT/bench_$V.json | head -1)"
done
