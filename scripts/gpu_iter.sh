#!/usr/bin/env bash
# One build -> measure iteration on the GPU box: a parity subset, then short
# benches of the env-selected variants (VAR / VALUES), then old-vs-new A/B
# against abtest/ when it exists.
# Usage: PYTEST_K="tiled" VAR=ROTOR_WRING VALUES="82 44" bash scripts/gpu_iter.sh <tag>
set -u
TAG=${1:-it}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { tail -30 "$OUT/build.log"; exit 1; }
if [ -n "${PYTEST_K:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > "$OUT/pytest.log" 2>&1
  echo "pytest rc=$? $(tail -1 "$OUT/pytest.log")"; grep -E "Error|assert" "$OUT/pytest.log" | head -5
fi
for V in ${VALUES:-default}; do
  if [ "$V" = default ]; then E=""; else E="${VAR}=$V"; fi
  env $E timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_$V.json" 2> "$OUT/bench_$V.err"
  python - "$OUT/bench_$V.json" "$E" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]; w = d.get("work") or {}
    print(sys.argv[2] or "default", "solve %.2f ms  fill %.2f  middle %.2f  frac %.3f" % (d["ms_per_step"], d["fill_ms"], r.get("middle_ms_per_step", 0), r["frac"]),
          " coarse_pass/visits %.3f quads %.3g exact %.3g" % ((w.get("middle_coarse_bound_evals", 0) / 32 / max(1, w.get("middle_split_visits", 1)) - 1) / 4, w.get("middle_filter_compares", 0), w.get("middle_exact_candidates", 0)) if w else "",
          " cycles " + " ".join("%s %.2f" % (k, v / max(1, sum(w["middle_warp_cycles"].values()))) for k, v in w["middle_warp_cycles"].items()) + " imbalance %.3f" % w.get("middle_warp_imbalance", 0) if w.get("middle_warp_cycles") else "")
except Exception as e:
    print(sys.argv[2], "bench failed", e, open(sys.argv[1].replace(".json", ".err")).read()[-800:])
PY
done
if [ -d abtest ] && [ -z "${NOAB:-}" ]; then
  for v in old new old; do
    if [ $v = old ]; then (cd abtest && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ../$OUT/ab_$v.json 2>&1)
    else timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ab_$v.json 2>&1; fi
    echo "ab $v $(grep -o '"ms_per_step": [0-9.]*' $OUT/ab_$v.json | head -1) $(grep -o '"middle_ms_per_step": [0-9.]*' $OUT/ab_$v.json)"
  done
fi
