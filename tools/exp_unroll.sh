# C4: rows in flight per warp in lz_proj (SDB_PROJ_UNROLL), then basis vectors per load batch in lz_update (SDB_UPD_TU), interleaved
cp paper_1308_5467_b200/libspecdens_b200.so /tmp/main.so
for v in t2 main t8 t16 t2 main t8; do
  if [ $v = main ]; then cp /tmp/main.so paper_1308_5467_b200/libspecdens_b200.so; else cp exp_lib/lib_$v.so paper_1308_5467_b200/libspecdens_b200.so; fi
  timeout 300 python tools/config_bench.py C4 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['seconds'],4), round(d['frac_vs_minimal_bytes'],3))"
done
cp /tmp/main.so paper_1308_5467_b200/libspecdens_b200.so
