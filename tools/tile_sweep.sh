cp paper_1308_5467_b200/libspecdens_b200.so /tmp/lib_orig.so
for nt in 512 1024; do
  cp tools/variants/lib_nt$nt.so paper_1308_5467_b200/libspecdens_b200.so
  for cfg in "16 2 1" "8 2 1" "8 2 2" "8 4 1" "16 2 2" "8 4 2"; do
    set -- $cfg
    SDB_TILE=1 SDB_TILE_CS=$1 SDB_TILE_TY=$2 SDB_TILE_PD=$3 python tools/config_bench.py C2 C5 --reps 2 2>/dev/null | python -c "import sys,json; [print(\"nt=$nt cs=$1 ty=$2 pd=$3\", d[\"config\"], round(d[\"step_us\"],1), round(d[\"frac_of_peak\"],3)) for d in map(json.loads, sys.stdin)]"
  done
done
cp /tmp/lib_orig.so paper_1308_5467_b200/libspecdens_b200.so
