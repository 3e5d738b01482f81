#!/usr/bin/env bash
# ncu evidence for one kernel configuration: launch list of one solve + full captures.
# Usage: gpurun -- bash scripts/gpu_profile.sh <tag> <kernel> "<regex:skip> ..."
set -u
TAG=${1:-p}; KERNEL=${2:-tiled}; CAPS=${3:-"k_tile_middle:14 k_tile_dep:16"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
ROTOR_KERNEL=$KERNEL timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$OUT/ncu_launches.log" 2>&1
echo "launches rc=$?"
python scripts/ncu_summary.py launches "$OUT/launches.csv"
for cap in $CAPS; do
  K=${cap%%:*}; SK=${cap##*:}
  ROTOR_KERNEL=$KERNEL timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s "$SK" -c 1 \
      -o "$OUT/full_$K" python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$OUT/ncu_full_$K.log" 2>&1
  echo "full $K rc=$?"
done
