#!/usr/bin/env bash
# Round-2 ncu evidence: launch list of one default (tile-DAG) config-4 solve,
# full captures of the middle / leaf / sub-product (diagonal schedule: one
# launch per tile diagonal, so -s picks a diagonal) and of k_batch (config 5).
# Usage: gpurun -- bash scripts/gpu_profile_r02.sh <tag>
set -u
TAG=${1:-p2}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" $B > "$OUT/ncu_launches.log" 2>&1
echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches_diag.csv" $B --schedule diagonal > "$OUT/ncu_launches_diag.log" 2>&1
echo "launches (diagonal) rc=$?"
for cap in ${CAPS:-k_tile_middle_wide:14 k_sub_leaf_row:100 k_sub_product_async:90}; do
  K=${cap%%:*}; SK=${cap##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s "$SK" -c 1 \
      -o "$OUT/full_$K" $B --schedule diagonal > "$OUT/ncu_full_$K.log" 2>&1
  echo "full $K rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_batch" -c 1 \
    -o "$OUT/full_k_batch" python bench.py --config 5 --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_full_k_batch.log" 2>&1
echo "full k_batch rc=$?"
