#!/usr/bin/env bash
# ncu evidence of exactly one config-4 solve per schedule (scripts/one_solve.py),
# plus full captures of the middle (diagonal schedule, -s 14: tile diagonal 16),
# the leaf and the sub-product.  Usage: gpurun -- bash scripts/gpu_profile_r02b.sh <tag>
set -u
TAG=${1:-p3}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { cat "$OUT/build.log"; exit 1; }
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for SCH in diagonal dag; do
  timeout 1500 ncu $M --log-file "$OUT/launches_$SCH.csv" python scripts/one_solve.py $SCH > "$OUT/ncu_launches_$SCH.log" 2>&1
  echo "launches $SCH rc=$?"
done
for cap in ${CAPS:-k_tile_middle_wide:14 k_sub_leaf_row:100 k_sub_product_async:90}; do
  K=${cap%%:*}; SK=${cap##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s "$SK" -c 1 \
      -o "$OUT/full_$K" python scripts/one_solve.py diagonal > "$OUT/ncu_full_$K.log" 2>&1
  echo "full $K rc=$?"
done
