#!/usr/bin/env bash
# Quick GPU iteration: build, microbench, tiled parity subset, short bench.
set -u
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
if [ -n "${MICRO:-}" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_minplus.cu && timeout 120 /tmp/mb > "$OUT/microbench.txt" 2>&1
  cat "$OUT/microbench.txt"
fi
timeout 900 python -m pytest tests -m gpu -x -q -rs ${PYTEST_K:+-k "$PYTEST_K"} > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?"; tail -15 "$OUT/pytest_gpu.log"
if [ -z "${NOBENCH:-}" ]; then
  for K in ${KERNELS:-tiled}; do
    ROTOR_KERNEL=$K timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > "$OUT/bench_$K.json" 2> "$OUT/bench_$K.err"
    echo "bench $K rc=$?"; cat "$OUT/bench_$K.json"; tail -3 "$OUT/bench_$K.err"
  done
fi
