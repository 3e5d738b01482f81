#!/usr/bin/env bash
# One GPU session of round evidence: tests + smoke + bench lines (gpu_round.sh),
# ncu launch lists of one solve per schedule + full captures (gpu_profile_r02b.sh),
# a tile-DAG timeline (ROTOR_TRACE), sanitizers.  Usage: gpurun -- bash scripts/gpu_evidence.sh <tag>
set -u
TAG=${1:-ev}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
bash scripts/gpu_round.sh "$TAG" tests,smoke,bench
bash scripts/gpu_profile_r02b.sh "$TAG/prof"
ROTOR_TRACE="$OUT/dag_trace.csv" timeout 300 python scripts/time_solve.py dag 2 > "$OUT/trace.log" 2>&1; echo "trace rc=$?"
if [ -n "${SAN:-}" ]; then bash scripts/sanitize.sh "$TAG/san" 2>&1 | tail -4; fi  # compute-sanitizer is closed on this pool
