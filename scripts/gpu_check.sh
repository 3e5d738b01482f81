#!/usr/bin/env bash
# One GPU session: parity tests, smoke, bench, ncu launch list and one full capture.
# Usage (from this container): gpurun --timeout 2400 -- bash scripts/gpu_check.sh [tag] [kernel] [what]
#   what: comma list of {tests,smoke,bench,ncu} (default all)
set -u
TAG=${1:-r01}
KERNEL=${2:-auto}
WHAT=${3:-tests,smoke,bench,ncu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
has() { [[ ",$WHAT," == *",$1,"* ]]; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rs > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest gpu rc=$?" | tee -a "$OUT/summary.txt"; tail -5 "$OUT/pytest_gpu.log"
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke rc=$?" | tee -a "$OUT/summary.txt"; tail -3 "$OUT/smoke.log"
fi
if has bench; then
  ROTOR_KERNEL=$KERNEL timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench rc=$?" | tee -a "$OUT/summary.txt"; cat "$OUT/bench.json"; tail -3 "$OUT/bench.err"
fi
if has ncu; then
  # launch list of one solve (cold-cache, serialised: compare shares, not absolutes)
  ROTOR_KERNEL=$KERNEL timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
      > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?" | tee -a "$OUT/summary.txt"
  # one full capture of the dominant kernel at a mid diagonal
  KREGEX=${KREGEX:-k_diag}
  KSKIP=${KSKIP:-500}
  ROTOR_KERNEL=$KERNEL timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" \
      -s "$KSKIP" -c 1 -o "$OUT/prof_full" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
      > "$OUT/ncu_full.log" 2>&1
  echo "ncu full rc=$?" | tee -a "$OUT/summary.txt"
fi
cat "$OUT/summary.txt"
