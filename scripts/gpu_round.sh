#!/usr/bin/env bash
# One GPU session for a round's evidence: parity tests, smoke, bench (N=1),
# ncu launch list with DRAM bytes, one full capture of the dominant kernel,
# compute-sanitizer passes.
# Usage: gpurun --timeout 2400 -- bash scripts/gpu_round.sh <tag> [what] (what: tests,smoke,bench,ncu,san)
set -u
TAG=${1:-r}
WHAT=${2:-tests,smoke,bench,ncu,san}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
has() { [[ ",$WHAT," == *",$1,"* ]]; }
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { tail -20 "$OUT/build.log"; exit 1; }
if has tests; then
  timeout 900 python -m pytest tests -m gpu -x -q -rs > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest gpu rc=$? $(tail -1 "$OUT/pytest_gpu.log")"
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke rc=$?"; tail -2 "$OUT/smoke.log"
fi
if has bench; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench rc=$?"; cut -c1-300 "$OUT/bench.json"
  timeout 600 python bench.py --config 5 > "$OUT/bench_cfg5.json" 2> "$OUT/bench_cfg5.err"
  echo "bench cfg5 rc=$?"; cut -c1-200 "$OUT/bench_cfg5.json"
  timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
  echo "bench reference rc=$?"; cut -c1-200 "$OUT/bench_reference.json"
fi
if has ncu; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?"
  for cap in ${CAPS:-k_tile_middle_wide:14 k_sub_leaf_row:100 k_sub_product_async:90}; do
    K=${cap%%:*}; SK=${cap##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s "$SK" -c 1 \
        -o "$OUT/full_$K" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$OUT/ncu_full_$K.log" 2>&1
    echo "ncu full $K rc=$?"
  done
fi
if has san; then
  bash scripts/sanitize.sh "$TAG/san" 2>&1 | tail -4
fi
if has sharded; then
  ROTOR_FORCE_SHARDED=1 timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench_sharded_1rank.json" 2> "$OUT/bench_sharded_1rank.err"
  echo "bench sharded (1 rank) rc=$?"; cut -c1-200 "$OUT/bench_sharded_1rank.json"
fi
