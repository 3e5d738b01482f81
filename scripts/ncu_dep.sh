set -u
OUT=gpurun_out/nd1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sub_leaf_row -s 6 -c 1 -o $OUT/leaf_d1 python scripts/one_solve.py diagonal > $OUT/ncu_leaf.log 2>&1; echo leaf rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sub_product -s 4 -c 1 -o $OUT/prod_d1 python scripts/one_solve.py diagonal > $OUT/ncu_prod.log 2>&1; echo prod rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_middle_wide -s 14 -c 1 -o $OUT/mid_d16 python scripts/one_solve.py diagonal > $OUT/ncu_mid.log 2>&1; echo mid rc=$?
